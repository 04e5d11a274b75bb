"""numpy/scipy restatement of the reference MO-FEM solve path (oracle only).

TEST INFRASTRUCTURE — see oracle/__init__.py for who may import this.

Dense q x q matrices throughout, exactly like the reference (fem1d.py:7-9):
operator application is a sum of dense GEMMs, the preconditioner inverse is a
pair of LU solves and the reduced solve uses LAPACK generalized ``eigh``.  The
functions are deliberately written in a flat functional style (dicts and
tuples instead of the reference's classes); each cites the reference lines it
restates.  Paths are relative to /root/reference/pkg/src/sylfem/.
"""

from __future__ import annotations

import math
import time
from collections import namedtuple

import numpy as np
import scipy.linalg as sla

__all__ = [
    "Domain", "unit_square", "cap_domain", "jar_domain", "wave_domain",
    "rect_domain", "DIRICHLET", "NEUMANN", "shape_tables", "dof_count",
    "dof_map", "assemble_dir", "assemble_lumped_dir", "direction_sets",
    "unit_degenerate", "prune_terms", "elliptic_terms", "parabolic_terms",
    "apply_terms", "precond_factors", "LUPrecond", "spectral_cache", "pcg_iterations",
    "reduced_solve", "mo_pcg", "imex_heat", "imex_rds", "dib_params",
    "dib_rates", "initial_fields", "full_node_grid", "expand_full",
    "interior", "seeded_modes", "OracleError", "pgm_bytes", "csv_text",
    "closed_form", "direct_solve", "perturbed_apply", "iteration_envelope",
]

DIRICHLET, NEUMANN = "dirichlet", "neumann"


class OracleError(Exception):
    """Raised where the reference raises (message text mirrors it)."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind  # reference exception class name


# ---------------------------------------------------------------------------
# domains (geometry.py:32-127): profile L(y), L'(y) and the x offset
# ---------------------------------------------------------------------------

Domain = namedtuple("Domain", "name L dL x_offset unit")


def unit_square():
    one = lambda s: np.ones_like(np.asarray(s, dtype=float))       # geometry.py:137-146
    zero = lambda s: np.zeros_like(np.asarray(s, dtype=float))
    return Domain("square", one, zero, 0.0, True)


def cap_domain():                                                   # geometry.py:148-151
    return Domain("cap", lambda s: 2.0 - np.asarray(s, float) ** 2,
                  lambda s: -2.0 * np.asarray(s, float), -0.5, False)


def jar_domain():                                                   # geometry.py:153-156
    return Domain("jar", lambda s: 2.0 + np.sin(2 * np.pi * np.asarray(s, float)),
                  lambda s: 2 * np.pi * np.cos(2 * np.pi * np.asarray(s, float)),
                  -0.5, False)


def wave_domain(amp=0.3):
    """x-normal domain 0 <= x <= 1 + amp sin(2 pi y)."""
    return Domain("wave", lambda s: 1.0 + amp * np.sin(2 * np.pi * np.asarray(s, float)),
                  lambda s: 2 * np.pi * amp * np.cos(2 * np.pi * np.asarray(s, float)),
                  0.0, False)


def rect_domain(width=2.0):
    """x-normal domain with constant profile L == width."""
    return Domain("rect", lambda s: width * np.ones_like(np.asarray(s, float)),
                  lambda s: np.zeros_like(np.asarray(s, float)), 0.0, False)


# ---------------------------------------------------------------------------
# 1D assembly (fem1d.py)
# ---------------------------------------------------------------------------

def shape_tables(k: int, nq: int):
    """Lagrange values/derivatives at mapped Gauss points (fem1d.py:37-73)."""
    nodes = np.linspace(0.0, 1.0, k + 1)
    g, gw = np.polynomial.legendre.leggauss(nq)
    xq, wq = 0.5 * (g + 1.0), 0.5 * gw
    psi = np.empty((k + 1, nq))
    dpsi = np.empty((k + 1, nq))
    for a in range(k + 1):
        others = [b for b in range(k + 1) if b != a]
        psi[a] = np.prod([(xq - nodes[b]) / (nodes[a] - nodes[b]) for b in others], axis=0) \
            if others else 1.0
        acc = np.zeros(nq)
        for c in others:
            term = np.full(nq, 1.0 / (nodes[a] - nodes[c]))
            for b in others:
                if b != c:
                    term = term * (xq - nodes[b]) / (nodes[a] - nodes[b])
            acc += term
        dpsi[a] = acc
    return xq, wq, psi, dpsi


def _check_basis(k, N):                                             # fem1d.py:90-98
    if not 1 <= k <= 4:
        raise OracleError("AssemblyError", f"degree must be in 1..4, got {k}")
    if N < 2:
        raise OracleError("AssemblyError", f"need at least 2 subintervals, got {N}")
    if N % k:
        raise OracleError("AssemblyError",
                          f"subinterval count {N} is not divisible by degree {k}")


def dof_count(N, bc):                                               # fem1d.py:32-34
    return N - 1 if bc == DIRICHLET else N + 1


def dof_map(N, bc):                                                 # fem1d.py:123-132
    m = np.arange(N + 1)
    if bc == DIRICHLET:
        m = m - 1
        m[0] = m[-1] = -1
    return m


def _add_local(mat, loc, rows, cols):
    """Scatter a local block, skipping trimmed (-1) rows/cols (fem1d.py:240-243)."""
    rk, ck = rows >= 0, cols >= 0
    mat[np.ix_(rows[rk], cols[ck])] += loc[np.ix_(rk, ck)]


def assemble_dir(k, N, bc, L, dL, offset=0.0, nq=None):
    """All weighted 1D matrices of one direction (fem1d.py:246-308)."""
    _check_basis(k, N)
    nq = max(k + 2, 5) if nq is None else nq                        # fem1d.py:134-137
    xq, wq, psi, dpsi = shape_tables(k, nq)
    h = k / N
    q = dof_count(N, bc)
    dm = dof_map(N, bc)
    names = ("A", "M", "B1", "B2", "C1", "C2", "M1", "M2", "M3")
    out = {n: np.zeros((q, q)) for n in names}
    out["M_full"] = np.zeros((q, N + 1))
    out["M3_full"] = np.zeros((q, N + 1))
    for e in range(N // k):
        xg = (e + xq) * h
        w = np.asarray(L(xg), dtype=float)
        if np.any(w <= 0.0):
            raise OracleError("GeometryError", f"profile nonpositive inside element {e}")
        dw = np.asarray(dL(xg), dtype=float)
        c = xg + offset
        glob = e * k + np.arange(k + 1)
        d = dm[glob]
        stiff = lambda wt: (dpsi * (wq * wt)) @ dpsi.T / h
        mass = lambda wt: (psi * (wq * wt)) @ psi.T * h
        _add_local(out["A"], stiff(np.ones_like(w)), d, d)
        _add_local(out["B1"], stiff(w), d, d)
        _add_local(out["B2"], stiff(c * c), d, d)
        _add_local(out["M"], mass(np.ones_like(w)), d, d)
        _add_local(out["M1"], mass(1.0 / w), d, d)
        _add_local(out["M2"], mass(dw * dw / w), d, d)
        _add_local(out["M3"], mass(w), d, d)
        _add_local(out["C1"], (dpsi * (wq * c)) @ psi.T, d, d)
        _add_local(out["C2"], (dpsi * (wq * dw)) @ psi.T, d, d)
        _add_local(out["M_full"], mass(np.ones_like(w)), d, glob)
        _add_local(out["M3_full"], mass(w), d, glob)
    return out


def assemble_lumped_dir(N, bc, L, dL, offset=0.0):
    """Lumped P1 matrices of one direction (fem1d.py:311-349)."""
    h = 1.0 / N
    q = dof_count(N, bc)
    dm = dof_map(N, bc)
    xs = np.arange(N + 1) / N
    w = np.asarray(L(xs), dtype=float)
    if np.any(w <= 0.0):
        raise OracleError("GeometryError", "profile nonpositive at a mesh node")
    dw = np.asarray(dL(xs), dtype=float)
    c = xs + offset
    out = {n: np.zeros((q, q)) for n in ("M0", "C", "A1", "A2")}
    lap = np.array([[1.0, -1.0], [-1.0, 1.0]])
    conv = np.array([[-0.5, -0.5], [0.5, 0.5]])
    for e in range(N):
        d = dm[[e, e + 1]]
        _add_local(out["M0"], np.diag([h / 2, h / 2]), d, d)
        _add_local(out["C"], conv, d, d)
        _add_local(out["A1"], lap * (w[e] + w[e + 1]) / (2 * h), d, d)
        _add_local(out["A2"], lap * (c[e] ** 2 + c[e + 1] ** 2) / (2 * h), d, d)
    keep = dm >= 0
    out["D1"] = np.diag(w[keep])
    out["D2"] = np.diag(dw[keep])
    out["D3"] = np.diag(c[keep])
    return out


def direction_sets(dom: Domain, k, n_sub, bc, lumped=False):
    """(x, y) direction dicts (fem1d.py:365-390): x carries the coordinate
    weights with the domain offset, y the profile weights."""
    nx, ny = (n_sub, n_sub) if np.isscalar(n_sub) else (int(n_sub[0]), int(n_sub[1]))
    one = unit_square()
    sets = []
    for n, (L, dL, off) in ((nx, (one.L, one.dL, dom.x_offset)), (ny, (dom.L, dom.dL, 0.0))):
        s = {"k": k, "N": n, "bc": bc, "q": dof_count(n, bc),
             "mats": assemble_dir(k, n, bc, L, dL, off)}
        if lumped:
            if k != 1:
                raise OracleError("AssemblyError", "lumped assembly supports degree-1 elements only")
            s["lumped"] = assemble_lumped_dir(n, bc, L, dL, off)
        sets.append(s)
    return sets[0], sets[1]


# ---------------------------------------------------------------------------
# grids (operators.py:39-73)
# ---------------------------------------------------------------------------

def full_node_grid(dom: Domain, x, y):
    xr = np.arange(x["N"] + 1) / x["N"] + dom.x_offset
    yr = np.arange(y["N"] + 1) / y["N"]
    X = np.asarray(dom.L(yr), float)[:, None] * xr[None, :]
    return X, np.broadcast_to(yr[:, None], X.shape).copy()


def expand_full(U, x, y):
    full = np.zeros((y["N"] + 1, x["N"] + 1))
    full[np.ix_(dof_map(y["N"], y["bc"]) >= 0, dof_map(x["N"], x["bc"]) >= 0)] = U
    return full


def interior(F, x, y):
    return np.asarray(F, float)[np.ix_(dof_map(y["N"], y["bc"]) >= 0,
                                       dof_map(x["N"], x["bc"]) >= 0)]


def _full_grid_check(F, x, y):                                     # operators.py:65-73
    F = np.asarray(F, dtype=float)
    if F.shape != (y["N"] + 1, x["N"] + 1):
        raise OracleError("OperatorError", "nodal source must cover the full node grid")
    return F


# ---------------------------------------------------------------------------
# operators (operators.py:97-297)
# ---------------------------------------------------------------------------

def prune_terms(terms):
    """Drop terms with an (almost) zero factor and validate (operators.py:100-119)."""
    kept = [(np.asarray(G, float), np.asarray(H, float)) for G, H in terms]
    kept = [(G, H) for G, H in kept
            if np.max(np.abs(G)) > 1e-15 and np.max(np.abs(H)) > 1e-15]
    if not kept:
        raise OracleError("OperatorError", "operator has no nonzero terms")
    qy, qx = kept[0][0].shape[0], kept[0][1].shape[0]
    if any(G.shape != (qy, qy) or H.shape != (qx, qx) for G, H in kept):
        raise OracleError("OperatorError", "inconsistent term factor shapes")
    return kept


def apply_terms(terms, U):
    """sum_t G_t U H_t, accumulated in term order (operators.py:124-131)."""
    out = np.zeros((terms[0][0].shape[0], terms[0][1].shape[0]))
    for G, H in terms:
        out += G @ U @ H
    return out


def unit_degenerate(y):                                             # operators.py:158-165
    m = y["mats"]
    s = max(np.max(np.abs(m["A"])), 1.0)
    return bool(np.max(np.abs(m["M2"])) <= 1e-14 * s and np.max(np.abs(m["C2"])) <= 1e-14 * s
                and np.max(np.abs(m["B1"] - m["A"])) <= 1e-13 * s
                and np.max(np.abs(m["M1"] - m["M"])) <= 1e-13
                and np.max(np.abs(m["M3"] - m["M"])) <= 1e-13)


def _lumped_rows(y):
    ly = y["lumped"]
    d1 = np.diag(ly["D1"])
    return ly, d1, ly["M0"] * d1


def elliptic_terms(x, y, gamma=0.0, lumped=False):
    """Term list + rhs map of -Lap + gamma (operators.py:177-234)."""
    if gamma < 0:
        raise OracleError("OperatorError", "reaction coefficient must be nonnegative")
    if x["bc"] == NEUMANN and gamma == 0.0:
        raise OracleError("OperatorError",
                          "singular operator: pure Neumann Laplacian needs gamma > 0")
    mx, my = x["mats"], y["mats"]
    if lumped:
        lx = x["lumped"]
        ly, d1, ml = _lumped_rows(y)
        terms = [(ly["M0"] / d1[:, None], mx["A"]),
                 (ly["A1"] + gamma * ml, lx["M0"]),
                 (np.diag(np.diag(ly["D2"]) ** 2 / d1) @ ly["M0"], lx["A2"]),
                 (-ly["D2"] @ ly["C"].T, lx["D3"] @ lx["C"].T),
                 (-ly["C"] @ ly["D2"], lx["C"] @ lx["D3"])]
        return prune_terms(terms), lambda F: ml @ interior(_full_grid_check(F, x, y), x, y) @ lx["M0"]
    if unit_degenerate(y):
        terms = [(my["A"] + 0.5 * gamma * my["M"], mx["M"]),
                 (my["M"], mx["A"] + 0.5 * gamma * mx["M"])]
    else:
        terms = [(my["M1"], mx["A"]), (my["B1"] + gamma * my["M3"], mx["M"]),
                 (my["M2"], mx["B2"]), (-my["C2"], mx["C1"]), (-my["C2"].T, mx["C1"].T)]
    return prune_terms(terms), lambda F: my["M3_full"] @ _full_grid_check(F, x, y) @ mx["M_full"].T


def parabolic_terms(x, y, d_u, tau, lumped=False):
    """Implicit-Euler step operator and its rhs map (operators.py:237-284)."""
    if d_u <= 0:
        raise OracleError("OperatorError", "diffusion coefficient must be positive")
    if tau < 0:
        raise OracleError("OperatorError", "timestep must be nonnegative")
    mx, my = x["mats"], y["mats"]
    c = d_u * tau
    if lumped:
        lx = x["lumped"]
        ly, d1, ml = _lumped_rows(y)
        terms = [(ml + c * ly["A1"], lx["M0"]),
                 (c * ly["M0"] / d1[:, None], mx["A"]),
                 (c * np.diag(np.diag(ly["D2"]) ** 2 / d1) @ ly["M0"], lx["A2"]),
                 (-c * ly["D2"] @ ly["C"].T, lx["D3"] @ lx["C"].T),
                 (-c * ly["C"] @ ly["D2"], lx["C"] @ lx["D3"])]
        return prune_terms(terms), lambda W: ml @ interior(_full_grid_check(W, x, y), x, y) @ lx["M0"]
    terms = [(my["M3"] + c * my["B1"], mx["M"]), (c * my["M1"], mx["A"]),
             (c * my["M2"], mx["B2"]), (-c * my["C2"], mx["C1"]),
             (-c * my["C2"].T, mx["C1"].T)]
    return prune_terms(terms), lambda W: my["M3_full"] @ _full_grid_check(W, x, y) @ mx["M_full"].T


# ---------------------------------------------------------------------------
# preconditioner (solvers.py:90-196)
# ---------------------------------------------------------------------------

def _rcond_check(mat, name):                                        # solvers.py:90-100
    try:
        cnd = np.linalg.cond(mat, 1)
    except np.linalg.LinAlgError:
        cnd = np.inf
    rc = 1.0 / cnd if np.isfinite(cnd) else 0.0
    if rc < 1e-14:
        raise OracleError("SolverError", f"preconditioner factor '{name}' is numerically "
                          f"singular (rcond ~ {rc:.2e})")


class LUPrecond:
    """U -> P_L^-1 U P_R^-1 by two dense LU solves (solvers.py:103-143)."""

    def __init__(self, left=None, right=None, lname="P_L", rname="P_R"):
        self.left, self.right, self.names = left, right, (lname, rname)
        self._lu = [None, None]
        for i, (m, n) in enumerate(((left, lname), (right, rname))):
            if m is not None:
                _rcond_check(m, n)
                self._lu[i] = sla.lu_factor(m)

    @property
    def identity(self):
        return self.left is None and self.right is None

    def inverse(self, R):
        if self.identity:
            return np.array(R, copy=True)
        Z = np.asarray(R)
        if self._lu[0] is not None:
            Z = sla.lu_solve(self._lu[0], Z)
        if self._lu[1] is not None:
            Z = sla.lu_solve(self._lu[1], Z.T, trans=1).T
        return Z


def precond_factors(kind, x, y, d_u=1.0, tau=0.0, lumped=False):
    """(left, right, left_name, right_name) of a named kind (solvers.py:156-196)."""
    if kind == "identity":
        return None, None, "identity", "identity"
    if kind == "parabolic_lumped":
        kind, lumped = "parabolic", True
    mx, my = x["mats"], y["mats"]
    if lumped and ("lumped" not in x or "lumped" not in y):
        raise OracleError("SolverError", "lumped preconditioner requested without lumped matrices")
    flat = unit_degenerate(y)
    if kind == "elliptic_square":
        return my["A"], mx["A"], "A(y)", "A(x)"
    if kind == "elliptic_xnormal":
        if lumped:
            r = mx["A"] if flat else mx["A"] + x["lumped"]["A2"]
            return y["lumped"]["A1"], r, "A1(y)", "A(x)" if flat else "A+A2(x)"
        r = mx["A"] if flat else mx["A"] + mx["B2"]
        return my["B1"], r, "B1(y)", "A(x)" if flat else "A+B2(x)"
    if kind == "parabolic":
        c = d_u * tau
        if lumped:
            ly, lx = y["lumped"], x["lumped"]
            left = ly["M0"] @ ly["D1"] + c * ly["A1"]
            right = lx["M0"] + c * (mx["A"] if flat else mx["A"] + lx["A2"])
            return left, right, "M0*D1+d*tau*A1(y)", "M0+d*tau*(A+A2)(x)"
        left = my["M3"] + c * my["B1"]
        right = mx["M"] + c * (mx["A"] if flat else mx["A"] + mx["B2"])
        return left, right, "M3+d*tau*B1(y)", "M+d*tau*(A+B2)(x)"
    raise OracleError("SolverError", f"unknown preconditioner kind '{kind}'")


# ---------------------------------------------------------------------------
# spectral reduction (solvers.py:203-300)
# ---------------------------------------------------------------------------

def _sign_fix(V):                                                   # solvers.py:203-208
    s = np.sign(V[np.argmax(np.abs(V), axis=0), np.arange(V.shape[1])])
    s[s == 0] = 1.0
    return V * s


def spectral_cache(terms):
    """Generalized eigh of both pencils with the term-order swap (solvers.py:256-281)."""
    if len(terms) != 2:
        raise OracleError("SolverError",
                          f"spectral reduction needs a two-term operator, got {len(terms)} terms")
    err = None
    for first, second, swapped in ((0, 1, False), (1, 0, True)):
        (G1, H1), (G2, H2) = terms[first], terms[second]
        try:
            l1, P1 = sla.eigh(G1, G2)
            l2, P2 = sla.eigh(H2, H1)
        except (np.linalg.LinAlgError, sla.LinAlgError) as exc:
            err = exc
            continue
        return {"lam1": l1, "lam2": l2, "P1": _sign_fix(P1), "P2": _sign_fix(P2),
                "swapped": swapped}
    raise OracleError("SolverError", f"operator is not reducible to Z1 U + U Z2 form: {err}")


def reduced_solve(terms, rhs, cache=None):
    """P1 [(P1^T B P2) / (lam1_i + lam2_j)] P2^T and its relative residual
    (solvers.py:245-253, 284-300)."""
    cache = spectral_cache(terms) if cache is None else cache
    den = cache["lam1"][:, None] + cache["lam2"][None, :]
    if np.min(np.abs(den)) < 1e-12:
        raise OracleError("SolverError", "spectral pencils are (numerically) singular")
    rhs = np.asarray(rhs, float)
    P1, P2 = cache["P1"], cache["P2"]
    U = P1 @ ((1.0 / den) * (P1.T @ rhs @ P2)) @ P2.T
    rel = np.linalg.norm(apply_terms(terms, U) - rhs) / max(np.linalg.norm(rhs), 1e-300)
    return U, rel, cache


def closed_form(gamma, f_int, N):
    """k = 1 Dirichlet unit square without an eigensolver (solvers.py:303-354):
    eigenvalues ((12N^2-g) l + 6Ng) / (12N - 2l), l = 2N(1-cos(i pi/N)), and
    the sine basis X with X^-1 = (2/N) X.  Returns (U, spectral residual)."""
    f_int = np.asarray(f_int, float)
    i = np.arange(1, N)
    la = 2.0 * N * (1.0 - np.cos(i * np.pi / N))
    lam = ((12.0 * N * N - gamma) * la + 6.0 * N * gamma) / (12.0 * N - 2.0 * la)
    den = lam[:, None] + lam[None, :]
    X = np.sin(np.outer(i, i) * np.pi / N)
    c = 2.0 / N
    fh = c * (X @ f_int @ X)
    U = c * (X @ (fh / den) @ X)
    return U, np.linalg.norm(den * (c * (X @ U @ X)) - fh) / max(np.linalg.norm(fh), 1e-300)


def direct_solve(terms, rhs):
    """The vec-form system sum_t G_t (x) H_t^T (row-major vec) solved densely
    (solvers.py:524-554 solves the same system by sparse LU)."""
    K = sum(np.kron(G, H.T) for G, H in terms)
    rhs = np.asarray(rhs, float)
    return np.linalg.solve(K, rhs.ravel()).reshape(rhs.shape)


def perturbed_apply(terms, variant):
    """The operator map with one deliberate change of rounding (test-side
    envelope of SURVEY finding 6): "reassoc" evaluates G (U H) instead of
    (G U) H, "reverse" accumulates the terms in reverse order."""
    if variant == "reassoc":
        def A(U):
            out = np.zeros((terms[0][0].shape[0], terms[0][1].shape[0]))
            for G, H in terms:
                out += G @ (U @ H)
            return out
        return A
    if variant == "reverse":
        return lambda U: apply_terms(terms[::-1], U)
    raise ValueError(variant)


def _precond_forms(pre):
    """The same preconditioner Z = P_L^-1 R P_R^-1 in three algebraic forms:
    LU solves (the reference), Cholesky solves (the factorization the banded
    SPIKE form is built on) and explicit inverses (the dense-GEMM form of
    BASELINE's north star)."""
    forms = {"lu": pre.inverse}
    if pre.identity:
        return forms
    L, R = pre.left, pre.right
    cl = sla.cho_factor(L) if L is not None else None
    cr = sla.cho_factor(R) if R is not None else None

    def chol(X):
        Z = sla.cho_solve(cl, X) if cl is not None else np.array(X, copy=True)
        return sla.cho_solve(cr, Z.T).T if cr is not None else Z
    Li = np.linalg.inv(L) if L is not None else None
    Ri = np.linalg.inv(R) if R is not None else None

    def explicit(X):
        Z = Li @ X if Li is not None else np.array(X, copy=True)
        return Z @ Ri if Ri is not None else Z
    forms["cholesky"], forms["inverse"] = chol, explicit
    return forms


def iteration_envelope(terms, rhs, pinv=None, rule=("residual", 1e-10), u0=None, max_iter=1000, ulp_seeds=3):
    """The reference's iteration count and the range it spans under changes
    of rounding alone (SURVEY finding 6): (iterations, lo, hi) over
    (a) G (U H) instead of (G U) H, (b) reversed term order and (c) the rhs
    perturbed by ~1 ulp (relative N(0, eps) noise, `ulp_seeds` seeds), the
    latter for every algebraic form of the preconditioner (LU / Cholesky /
    explicit inverse, when ``pinv`` is an ``LUPrecond`` or its bound
    ``inverse``).  A faithful implementation lands within hi - lo (+1) of
    the reference's count."""
    pre = getattr(pinv, "__self__", pinv) if pinv is not None else None
    forms = _precond_forms(pre) if isinstance(pre, LUPrecond) else {"lu": pinv}
    rhs = np.asarray(rhs, float)

    def run(b, P, **kw):
        return mo_pcg(terms, b, P, rule, u0=u0, max_iter=max_iter, **kw)["iterations"]
    base = run(rhs, forms["lu"])
    its = [base] + [run(rhs, forms["lu"], apply=perturbed_apply(terms, v)) for v in ("reassoc", "reverse")]
    for P in forms.values():
        for sd in range(ulp_seeds):
            xi = np.random.default_rng(1000 + sd).standard_normal(rhs.shape)
            its.append(run(rhs * (1.0 + np.finfo(float).eps * xi), P))
    return base, min(its), max(its)


# ---------------------------------------------------------------------------
# MO-PCG (solvers.py:361-453)
# ---------------------------------------------------------------------------

_SMALL = 512 * 512
_ONE = {"depth": 0}


class _one_thread:
    """Single-threaded BLAS for small grids (re-entrant; no-op without threadpoolctl)."""

    def __enter__(self):
        self.ctx = None
        if _ONE["depth"] == 0:
            try:
                from threadpoolctl import threadpool_limits
                self.ctx = threadpool_limits(limits=1)
            except ImportError:
                pass
        _ONE["depth"] += 1
        return self

    def __exit__(self, *exc):
        _ONE["depth"] -= 1
        if self.ctx is not None:
            self.ctx.unregister()


def mo_pcg(terms, rhs, pinv=None, rule=("residual", 1e-10), u0=None,
           max_iter=1000, record=False, apply=None):
    """Matrix-oriented PCG with the reference's recurrences and stop logic.

    ``pinv`` maps R -> Z (identity copy when None); ``rule`` is
    ("residual", tol) or ("increment", threshold).  Returns a dict with
    solution, iterations, history, increments, reason, iterates, wall.
    ``apply`` overrides the operator map (used for the CPU baseline timing
    of alternative operator evaluations).
    """
    rhs = np.asarray(rhs, float)
    if rhs.size < _SMALL and _ONE["depth"] == 0:  # many tiny GEMMs: BLAS threads only add latency
        with _one_thread():
            return mo_pcg(terms, rhs, pinv, rule, u0, max_iter, record, apply)
    A = (lambda V: apply_terms(terms, V)) if apply is None else apply
    P = (lambda V: np.array(V, copy=True)) if pinv is None else pinv
    t0 = time.perf_counter()
    if u0 is None:
        U = np.zeros_like(rhs)
        R = rhs.copy()
    else:
        U = np.array(u0, dtype=float, copy=True)
        R = rhs - A(U)
    res0 = np.linalg.norm(R)
    hist, incs = [res0], []
    its = [U.copy()] if record else None
    out = lambda n, why: {"solution": U, "iterations": n, "history": np.asarray(hist),
                          "increments": np.asarray(incs), "reason": why, "iterates": its,
                          "wall": time.perf_counter() - t0}
    if res0 == 0.0:
        return out(0, "tolerance")
    Z = P(R)
    Q = Z.copy()
    rz = float(np.vdot(Z, R))
    for s in range(max_iter):
        W = A(Q)
        qw = float(np.vdot(W, Q))
        if qw <= 0.0:
            raise OracleError("OperatorError", "operator is not positive definite along a "
                              f"search direction (<L(Q), Q> = {qw:.3e} at iteration {s})")
        alpha = rz / qw
        U += alpha * Q
        R -= alpha * W
        res = np.linalg.norm(R)
        if not np.isfinite(res):
            raise OracleError("SolverError", f"mo_pcg residual became non-finite at iteration {s}")
        hist.append(res)
        incs.append(abs(alpha) * np.linalg.norm(Q))
        if record:
            its.append(U.copy())
        if rule[0] == "residual" and res <= rule[1] * res0:
            return out(s + 1, "tolerance")
        if rule[0] == "increment" and incs[-1] <= rule[1]:
            return out(s + 1, "increment")
        Z = P(R)
        rz_new = float(np.vdot(Z, R))
        beta = rz_new / rz
        rz = rz_new
        Q *= beta
        Q += Z
    return out(max_iter, "max_iter")


def pcg_iterations(terms, rhs, pinv, u0=None):
    """The MO-PCG loop of solvers.py:415-452 one iteration at a time, without
    a stop test: a generator whose first ``next()`` runs the setup part
    (solvers.py:389-420: R_0, Z_0, <Z_0,R_0>) and yields |R_0|, and every
    further ``next()`` runs one iteration and yields |R_s|.  The CPU-baseline
    timer of bench.py times the iterations individually.  Same arithmetic
    as ``mo_pcg``."""
    A = lambda V: apply_terms(terms, V)
    rhs = np.asarray(rhs, float)
    if u0 is None:
        U = np.zeros_like(rhs)
        R = rhs.copy()
    else:
        U = np.array(u0, dtype=float, copy=True)
        R = rhs - A(U)
    Z = pinv(R)
    Q = Z.copy()
    rz = float(np.vdot(Z, R))
    yield np.linalg.norm(R)
    while True:
        W = A(Q)
        alpha = rz / float(np.vdot(W, Q))
        U += alpha * Q
        R -= alpha * W
        res = np.linalg.norm(R)
        Z = pinv(R)
        rz_new = float(np.vdot(Z, R))
        beta = rz_new / rz
        rz = rz_new
        Q *= beta
        Q += Z
        yield res


# ---------------------------------------------------------------------------
# IMEX drivers (timestepping.py:28-220)
# ---------------------------------------------------------------------------

def n_steps(tau, t_final):                                          # timestepping.py:39-41
    return max(1, math.ceil(t_final / tau - 1e-9))


def _blowup(U):                                                     # timestepping.py:86-91
    return (not np.all(np.isfinite(U))) or np.max(np.abs(U)) > 1e100


def _stop_rule(rule, tol, tau):                                     # timestepping.py:54-59
    return ("residual", tau) if rule == "tau" else ("residual", tol)


def imex_heat(dom, x, y, d_u, source, u0, tau, t_final, rule="tau", tol=1e-10,
              max_iter=400, precond="auto", lumped=False):
    """u_t - d Lap u = source(u, X, Y, t) (timestepping.py:126-159)."""
    terms, rhs_of = parabolic_terms(x, y, d_u, tau, lumped)
    kind = ("parabolic_lumped" if lumped else "parabolic") if precond == "auto" else precond
    pre = LUPrecond(*precond_factors(kind, x, y, d_u=d_u, tau=tau, lumped=lumped))
    X, Y = full_node_grid(dom, x, y)
    U = np.array(u0, dtype=float, copy=True)
    n = n_steps(tau, t_final)
    incs, iters = np.empty(n), np.empty(n, dtype=int)
    for k in range(n):
        Uf = expand_full(U, x, y)
        W = Uf + tau * np.asarray(source(Uf, X, Y, k * tau), dtype=float)
        if _blowup(W):
            raise OracleError("BlowUpError", f"solution blew up at step {k} (species u)")
        r = mo_pcg(terms, rhs_of(W), pre.inverse, _stop_rule(rule, tol, tau), u0=U,
                   max_iter=max_iter)
        if r["reason"] == "max_iter":
            raise OracleError("SolverError", f"inner PCG did not converge in {max_iter} iterations")
        if _blowup(r["solution"]):
            raise OracleError("BlowUpError", f"solution blew up at step {k} (species u)")
        incs[k] = np.linalg.norm(r["solution"] - U)
        iters[k] = r["iterations"]
        U = r["solution"]
    return {"final": U, "increments": incs, "iterations": iters,
            "times": (1 + np.arange(n)) * tau}


def imex_rds(x, y, d_u, d_v, kinetics, rho, state0, tau, t_final, rule="tau",
             tol=1e-10, max_iter=400, precond="auto", lumped=False,
             snapshot_every=0, steady_eps=1e-8):
    """Two-species IMEX Euler, explicit kinetics (timestepping.py:162-220)."""
    if d_u <= 0 or d_v <= 0 or rho <= 0:
        raise OracleError("ConfigError", "d_u, d_v and rho must be positive")
    if x["bc"] != NEUMANN:
        raise OracleError("ConfigError", "the reaction-diffusion stepper expects zero-flux BCs")
    f, g = kinetics
    tu, rhs_of = parabolic_terms(x, y, d_u, tau, lumped)
    tv, _ = parabolic_terms(x, y, d_v, tau, lumped)
    kind = ("parabolic_lumped" if lumped else "parabolic") if precond == "auto" else precond
    pu = LUPrecond(*precond_factors(kind, x, y, d_u=d_u, tau=tau, lumped=lumped))
    pv = LUPrecond(*precond_factors(kind, x, y, d_u=d_v, tau=tau, lumped=lumped))
    stop = _stop_rule(rule, tol, tau)
    U = np.array(state0[0], dtype=float, copy=True)
    V = np.array(state0[1], dtype=float, copy=True)
    n = n_steps(tau, t_final)
    incs, iters = np.empty((n, 2)), np.empty((n, 2), dtype=int)
    snaps, steady = [], None

    def solve(terms, pre, rhs, warm, k, sp):
        r = mo_pcg(terms, rhs, pre.inverse, stop, u0=warm, max_iter=max_iter)
        if r["reason"] == "max_iter":
            raise OracleError("SolverError", f"inner PCG did not converge in {max_iter} iterations")
        if _blowup(r["solution"]):
            raise OracleError("BlowUpError", f"solution blew up at step {k} (species {sp})")
        return r["solution"], r["iterations"]

    for k in range(n):
        fv, gv = f(U, V), g(U, V)
        Wu = U + tau * rho * np.asarray(fv)
        if _blowup(Wu):
            raise OracleError("BlowUpError", f"solution blew up at step {k} (species u)")
        Un, iu = solve(tu, pu, rhs_of(Wu), U, k, "u")
        Wv = V + tau * rho * np.asarray(gv)
        if _blowup(Wv):
            raise OracleError("BlowUpError", f"solution blew up at step {k} (species v)")
        Vn, iv = solve(tv, pv, rhs_of(Wv), V, k, "v")
        incs[k] = (np.linalg.norm(Un - U), np.linalg.norm(Vn - V))
        iters[k] = (iu, iv)
        U, V = Un, Vn
        if steady is None and np.all(incs[k] <= steady_eps * max(np.linalg.norm(U), 1e-300)):
            steady = k
        if snapshot_every and ((k + 1) % snapshot_every == 0 or k == n - 1):
            snaps.append((k + 1, U.copy(), V.copy()))
    return {"final": (U, V), "increments": incs, "iterations": iters,
            "times": (1 + np.arange(n)) * tau, "steady_step": steady, "snapshots": snaps}


# ---------------------------------------------------------------------------
# DIB kinetics and initial data (models.py:19-126)
# ---------------------------------------------------------------------------

def dib_params(alpha=0.5, gamma_k=0.2, A1=10.0, A2=30.0, B=25.0, C=7.0, D=None,
               k2=2.5, k3=1.5, d_theta=20.0, rho=400.0):
    """Parameter dict with D slaved to C when unset (models.py:19-28, 55-59)."""
    if D is None:
        D = C * (1 - alpha) * (1 - gamma_k * (1 - alpha)) / (alpha * (1 + gamma_k * alpha))
    return dict(alpha=alpha, gamma_k=gamma_k, A1=A1, A2=A2, B=B, C=C, D=D, k2=k2,
                k3=k3, d_theta=d_theta, rho=rho)


def dib_rates(eta, theta, p):
    """(f, g) of the electrodeposition model (models.py:74-82)."""
    eta, theta = np.asarray(eta, float), np.asarray(theta, float)
    f = p["A1"] * (1.0 - theta) * eta - p["A2"] * eta ** 3 - p["B"] * (theta - p["alpha"])
    g = (p["C"] * (1.0 + p["k2"] * eta) * (1.0 - theta) * (1.0 - p["gamma_k"] * (1.0 - theta))
         - p["D"] * theta * (1.0 + p["gamma_k"] * theta) * (1.0 + p["k3"] * eta))
    return f, g


def initial_fields(shape, amplitude=1e-4, seed=20240):
    """(0, 0.5) + amplitude * U[0,1) from Philox4x64 keyed by seed (models.py:103-126)."""
    gen = np.random.Generator(np.random.Philox(key=seed))
    eta = 0.0 + amplitude * gen.random(tuple(shape))
    theta = 0.5 + amplitude * gen.random(tuple(shape))
    return eta, theta


# ---------------------------------------------------------------------------
# seeded 8-mode sources of BASELINE.json
# ---------------------------------------------------------------------------

def seeded_modes(seed, n_modes=8):
    """a, b in 1..16 and N(0,1) amplitudes drawn in the order a, b, c."""
    rng = np.random.default_rng(seed)
    a = rng.integers(1, 17, n_modes)
    b = rng.integers(1, 17, n_modes)
    c = rng.standard_normal(n_modes)
    return a, b, c


# ---------------------------------------------------------------------------
# trajectory outputs (harness.py:424-491)
# ---------------------------------------------------------------------------

def pgm_bytes(array):
    """File bytes of harness.write_pgm (harness.py:475-491)."""
    a = np.asarray(array, dtype=float)
    lo, hi = float(np.min(a)), float(np.max(a))
    span = hi - lo
    if span > max(1e-12 * max(abs(hi), abs(lo)), 1e-14):
        scaled = np.round((a - lo) / span * 65535.0)
    else:
        scaled = np.zeros_like(a)
    return f"P5\n{a.shape[1]} {a.shape[0]}\n65535\n".encode() + scaled.astype(">u2").tobytes()


def csv_text(header, rows):
    """File text of harness.write_csv (harness.py:424-440): CRLF rows, repr floats."""
    import csv as _csv
    import io as _io

    def fmt(v):
        if isinstance(v, (float, np.floating)):
            return repr(float(v))
        if isinstance(v, (int, np.integer)):
            return str(int(v))
        return str(v)
    buf = _io.StringIO(newline="")
    w = _csv.writer(buf)
    w.writerow(header)
    for row in rows:
        w.writerow([fmt(v) for v in row])
    return buf.getvalue()
