"""Reduced (spectral) solve and MO-PCG on the B200 — drop-in for solvers.py.

Same entry points, report types, stopping rules, guards and error messages as
the reference (solvers.py:36-453).  What changes is where the work runs:

* ``Preconditioner.apply_inverse`` (solvers.py:134-143) — the reference does
  two dense LU solves.  Here the single-term preconditioner P_L U P_R is
  applied with FP64 DMMA tensor-core GEMMs: ``mode="inverse"`` (default) as
  Z = P_L^-1 R P_R^-1 with the dense inverses formed once on the device by
  banded Cholesky sweeps (2 GEMMs, 4 q^3 flops); ``mode="spectral"`` as
  V_L [(V_L^T R V_R) / (lam_i mu_j)] V_R^T (4 GEMMs); ``mode="banded"``
   as banded Cholesky sweeps, O(q^2 k).
* ``solve_reduced`` (solvers.py:284-300) — LAPACK generalized ``eigh`` on the
  host (the reference's route, off the loop), then the 4-GEMM spectral
  sandwich with the 1/(lam1_i + lam2_j) Hadamard fused into a GEMM epilogue.
* ``mo_pcg`` (solvers.py:365-453) — the whole loop is device resident (one
  CUDA-graph launch per solve; see csrc/solver.cu).
"""

from __future__ import annotations

import math
import os
import time
import weakref
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.linalg.lapack as lapack

from . import _native as nat
from .banded import Band
from .exceptions import OperatorError, SolverError
from .fem1d import DirectionSet
from .operators import SylvesterOperator, is_unit_degenerate, to_kronecker, unvec, vec

RCOND_GUARD = 1e-14
PENCIL_GUARD = 1e-12
DEFAULT_TOL = 1e-10
DEFAULT_MAX_ITER = 1000
PRECOND_MODES = ("inverse", "spectral", "banded")


def default_precond_mode() -> str:
    mode = os.environ.get("SYLFEM_B200_PRECOND", "inverse")
    if mode not in PRECOND_MODES:
        raise SolverError(f"SYLFEM_B200_PRECOND must be one of {PRECOND_MODES}, got '{mode}'")
    return mode


@dataclass
class SolveReport:
    """Solution plus convergence record of one linear solve (solvers.py:36-46)."""

    solution: object
    method: str
    iterations: int
    residual_history: np.ndarray
    stop_reason: str
    wall_time: float
    diagnostics: dict = field(default_factory=dict)


# ------------------------------------------------------------- stopping ----
@dataclass(frozen=True)
class StoppingRule:
    """Residual-relative or increment-absolute stop test (solvers.py:53-63)."""

    kind: str
    value: float

    def describe(self) -> str:
        if self.kind == "residual":
            return f"|R_s| <= {self.value:g} * |R_0|"
        if self.kind == "budget":
            return "fixed iteration budget (max_iter)"
        return f"|U_s+1 - U_s| <= {self.value:g}"

    @property
    def native_kind(self) -> int:
        return {"residual": nat.RULE_RESIDUAL, "increment": nat.RULE_INCREMENT,
                "budget": nat.RULE_BUDGET}[self.kind]


def relative_residual(tol: float = DEFAULT_TOL) -> StoppingRule:
    return StoppingRule("residual", float(tol))


def increment_threshold(threshold: float) -> StoppingRule:
    return StoppingRule("increment", float(threshold))


def reference_increment(reference_error_norm: float, fraction: float = 0.05) -> StoppingRule:
    return increment_threshold(fraction * reference_error_norm)


def timestep_residual(tau: float) -> StoppingRule:
    return relative_residual(tau)


def fixed_budget() -> StoppingRule:
    """No tolerance test: every solve runs exactly ``max_iter`` iterations and
    reports "max_iter" (fixed-work benchmarking, SURVEY §8 d; no reference
    counterpart).  Inside the IMEX drivers (``InnerSolver(rule="budget")``)
    reaching the budget completes the step instead of raising."""
    return StoppingRule("budget", 0.0)


# ------------------------------------------------------- preconditioner ----
def _lapack_band(m: Band):
    """LAPACK general-band storage (2kl+ku+1, n) of a square Band."""
    lo, hi = m.offsets()
    kl, ku = max(-lo, 0), max(hi, 0)
    n = m.shape[0]
    ab = np.zeros((2 * kl + ku + 1, n))
    c = m.sparse.tocoo()
    ab[kl + ku + c.row - c.col, c.col] = c.data
    return ab, kl, ku


def _rcond(mat) -> float:
    """1-norm reciprocal condition number: LAPACK's banded estimate for band
    factors, the exact value of the reference (np.linalg.cond(., 1),
    solvers.py:90-100) whenever the estimate lands within 100x of the guard
    (the estimate may overstate rcond) and for dense factors."""
    if isinstance(mat, Band) and mat.half_bandwidth() <= 16:
        ab, kl, ku = _lapack_band(mat)
        anorm = float(np.max(np.asarray(abs(mat.sparse).sum(axis=0)).ravel()))
        lu, ipiv, info = lapack.dgbtrf(ab, kl, ku)
        if info > 0:
            return 0.0
        rc, info = lapack.dgbcon(kl, ku, lu, ipiv, anorm)
        rc = float(rc) if np.isfinite(rc) else 0.0
        if rc > 100.0 * RCOND_GUARD:
            return rc
        mat = mat.toarray()
    try:
        c = np.linalg.cond(np.asarray(mat, dtype=float), 1)
    except np.linalg.LinAlgError:
        c = np.inf
    return 0.0 if not np.isfinite(c) else 1.0 / c


def _rcond_guard(mat, name: str) -> None:
    """solvers.py:90-100."""
    rc = _rcond(mat)
    if rc < RCOND_GUARD:
        raise SolverError(f"preconditioner factor '{name}' is numerically singular (rcond ~ {rc:.2e})")


def _as_factor(m):
    if m is None:
        return None
    if isinstance(m, Band):
        return m
    import scipy.sparse as sp
    if sp.issparse(m):
        return Band(m)
    return np.asarray(m, dtype=float)


def _cholesky_band(m, q: int):
    """Lower banded Cholesky in the device layout: band[i][d] = C[i][i-b+d],
    band[i][b] = 1 / C[i][i].  Returns (b, band) or None if not SPD-banded."""
    if m is None:
        return 0, np.ones((q, 1))
    b = m.half_bandwidth() if isinstance(m, Band) else None
    if b is None or b > 4:
        return None
    M = m.sparse
    if abs(M - M.T).max() > 1e-12 * max(m.max_abs(), 1e-300):
        return None
    ab = np.zeros((b + 1, q))  # LAPACK lower: ab[i-j, j] = A[i, j]
    c = M.tocoo()
    low = c.row >= c.col
    ab[c.row[low] - c.col[low], c.col[low]] = c.data[low]
    try:
        L = sla.cholesky_banded(ab, lower=True)
    except np.linalg.LinAlgError:
        return None
    band = np.zeros((q, b + 1))
    for d in range(b + 1):  # C[i][i-b+d] = L[b-d, i-(b-d)]
        off = b - d
        band[off:, d] = L[off, : q - off]
    band[:, b] = 1.0 / L[0, :]
    return b, band


def _sparse_of(m):
    return m.sparse.tocsr() if isinstance(m, Band) else sp.csr_matrix(np.asarray(m, dtype=float))


class KroneckerCSR(sp.csr_matrix):
    """csr_matrix of a Kronecker-structured preconditioner (as_kronecker)
    that carries the Preconditioner it was built from."""

    sfb_pre = None
    sfb_shape = None


def set_strassen_min_q(min_q: int) -> int:
    """Grid size from which the inverse-form preconditioner products (the two
    dense solves of solvers.py:134-143 as DMMA GEMMs) run as up to three
    Strassen levels (7 half-size products per level; odd shapes are padded
    with zeros inside the passes).  0 disables it.  Applies to device preconditioners built
    afterwards; returns the previous threshold (default 2000, or
    SYLFEM_B200_STRASSEN_MINQ)."""
    return int(nat.lib().sfb_set_strassen_min_q(int(min_q)))


def set_strassen_levels(levels: int) -> int:
    """Most Strassen levels taken by the inverse-form products (0..3, default
    3: q = 8192 runs 343 GEMMs of 1024^3 per product); returns the previous value."""
    return int(nat.lib().sfb_set_strassen_levels(int(levels)))


class Preconditioner:
    """Single-term preconditioner U -> P_L U P_R (solvers.py:103-150).

    The factors are kept as given (Band or dense); the device form is built on
    first use according to ``mode`` (see module docstring)."""

    def __init__(self, left=None, right=None, left_name: str = "P_L", right_name: str = "P_R",
                 mode: str | None = None):
        self.left = _as_factor(left)
        self.right = _as_factor(right)
        self.left_name = left_name
        self.right_name = right_name
        self.mode = default_precond_mode() if mode is None else mode
        if self.mode not in PRECOND_MODES:
            raise SolverError(f"unknown preconditioner mode '{self.mode}'")
        if self.left is not None:
            _rcond_guard(self.left, left_name)
        if self.right is not None:
            _rcond_guard(self.right, right_name)
        self._handle = None
        self._fwd = None
        self.shape = None if self.is_identity else (
            (self.left.shape[0] if self.left is not None else self.right.shape[0]),
            (self.right.shape[0] if self.right is not None else self.left.shape[0]))

    @property
    def is_identity(self) -> bool:
        return self.left is None and self.right is None

    def as_kronecker(self, shape) -> sp.csr_matrix:
        """Sparse vec-form matrix P_R^T (x) P_L (solvers.py:145-150), for the
        vector cross-check path.  The returned matrix remembers this
        preconditioner, so vector_pcg applies its inverse with the device
        kernels instead of a sparse factorisation."""
        qy, qx = shape
        left = sp.identity(qy, format="csr") if self.left is None else _sparse_of(self.left)
        right = sp.identity(qx, format="csr") if self.right is None else _sparse_of(self.right)
        K = KroneckerCSR(sp.kron(right.T.tocsr(), left, format="csr"))
        K.sfb_pre, K.sfb_shape = self, (qy, qx)
        return K

    # ---- device form -----------------------------------------------------
    def native(self, shape=None):
        """Device preconditioner for grids of ``shape`` (needed for identity)."""
        shape = tuple(shape) if shape is not None else self.shape
        if self._handle is not None and self._handle_shape == shape:
            return self._handle.p
        if shape is None:
            raise SolverError("identity preconditioner needs a grid shape")
        qy, qx = shape
        L = nat.lib()
        out = nat.C.c_void_p()
        if self.is_identity:
            nat.check(L.sfb_pre_create(qy, qx, nat.PRE_IDENTITY, None, None, None, None,
                                       nat.C.byref(out)), "preconditioner")
        elif self.mode == "banded":
            cl, cr = _cholesky_band(self.left, qy), _cholesky_band(self.right, qx)
            if cl is None or cr is None:
                raise SolverError("banded preconditioner mode needs symmetric positive definite "
                                  "factors with half-bandwidth <= 4")
            nat.check(L.sfb_pre_create_banded(qy, qx, cl[0], nat.host_ptr(np.ascontiguousarray(cl[1])),
                                              cr[0], nat.host_ptr(np.ascontiguousarray(cr[1])),
                                              nat.C.byref(out)), "preconditioner")
        elif self.mode == "spectral":
            lamL, VL = self._eigh(self.left, qy)
            lamR, VR = self._eigh(self.right, qx)
            nat.check(L.sfb_pre_create(qy, qx, nat.PRE_SPECTRAL_PROD, nat.host_ptr(VL), nat.host_ptr(VR),
                                       nat.host_ptr(lamL), nat.host_ptr(lamR), nat.C.byref(out)),
                      "preconditioner")
        else:
            # the inverses stay on the device (sfb_pre_create copies device to device)
            Linv = self._inverse(self.left, qy, left=True)
            RinvT = self._inverse(self.right, qx, left=False).T.contiguous()
            nat.check(L.sfb_pre_create(qy, qx, nat.PRE_INVERSE, nat.ptr(Linv), nat.ptr(RinvT),
                                       None, None, nat.C.byref(out)), "preconditioner")
            del Linv, RinvT
        self._handle = nat.Handle(out.value, L.sfb_pre_destroy)
        self._handle_shape = shape
        return self._handle.p

    def uses_strassen(self, shape=None) -> int:
        """Strassen levels the device form's dense products use (0: classic
        GEMMs; see set_strassen_min_q, set_strassen_levels)."""
        return int(nat.lib().sfb_pre_uses_strassen(self.native(shape)))

    @staticmethod
    def _eigh(m, q):
        if m is None:
            return np.ones(q), np.eye(q)
        A = np.asarray(m, dtype=float)
        # the reference solves with the factor itself (LU); the spectral form
        # is only the same preconditioner for a symmetric factor
        if np.max(np.abs(A - A.T)) > 1e-12 * max(np.max(np.abs(A)), 1e-300):
            raise SolverError("spectral preconditioner form needs symmetric factors; use mode='inverse'")
        lam, V = sla.eigh(0.5 * (A + A.T), driver="evd")
        return np.ascontiguousarray(lam), np.ascontiguousarray(V)

    @staticmethod
    def _inverse(m, q, left: bool):
        """Dense inverse as a CUDA tensor (setup, off the loop): device
        banded-Cholesky sweeps over the identity for SPD banded factors, host
        LAPACK otherwise.  It is never staged through the host on the banded
        route (2 x q^2 doubles per factor at q = 8192 would be 1 GB of copies)."""
        t = nat.torch()
        if m is None:
            return t.eye(q, dtype=t.float64, device="cuda")
        ch = _cholesky_band(m, q)
        if ch is None:
            return nat.to_device(np.linalg.inv(np.asarray(m, dtype=float)))
        L = nat.lib()
        one = np.ones((q, 1))
        out = nat.C.c_void_p()
        b = np.ascontiguousarray(ch[1])
        if left:  # P^-1 I by column sweeps
            rc = L.sfb_pre_create_banded(q, q, ch[0], nat.host_ptr(b), 0, nat.host_ptr(one), nat.C.byref(out))
        else:     # I P^-1 by row sweeps
            rc = L.sfb_pre_create_banded(q, q, 0, nat.host_ptr(one), ch[0], nat.host_ptr(b), nat.C.byref(out))
        nat.check(rc, "preconditioner inverse")
        h = nat.Handle(out.value, L.sfb_pre_destroy)
        eye = t.eye(q, dtype=t.float64, device="cuda")
        inv = t.empty_like(eye)
        nat.check(L.sfb_pre_apply(h.p, nat.ptr(eye), q, nat.ptr(inv), q, nat.stream()), "inverse")
        return inv

    # ---- application -----------------------------------------------------
    def apply(self, U):
        """P_L U P_R (solvers.py:124-132)."""
        if self.is_identity:
            return U.clone() if nat.is_device(U) else np.array(U, copy=True)
        if self._fwd is None:
            qy, qx = self.shape
            self._fwd = SylvesterOperator([(self.left if self.left is not None else Band.diag(np.ones(qy)),
                                            self.right if self.right is not None else Band.diag(np.ones(qx)))])
        return self._fwd.apply(U)

    def apply_inverse(self, U):
        """P_L^-1 U P_R^-1 (solvers.py:134-143)."""
        on_dev = nat.is_device(U)
        if self.is_identity:
            return U.clone() if on_dev else np.array(U, copy=True)
        t = nat.torch()
        Ud = nat.to_device(U)
        qy, qx = Ud.shape
        if self.shape != (qy, qx):
            raise OperatorError(f"grid shape {(qy, qx)} does not match preconditioner {self.shape}")
        Z = t.empty_like(Ud)
        nat.check(nat.lib().sfb_pre_apply(self.native(), nat.ptr(Ud), qx, nat.ptr(Z), qx, nat.stream()),
                  "apply_inverse")
        return Z if on_dev else nat.to_host(Z)


IDENTITY_PRECONDITIONER = "identity"


class TwoTermPreconditioner:
    """Opt-in preconditioner P(U) = G1 U H1 + G2 U H2 applied exactly in the
    spectral space of its two pencils (the north star's
    "(lambda_i + mu_j)" form): Z = P1 [(P1^T R P2) / (lam1_i + lam2_j)] P2^T,
    the same 4-GEMM DMMA sandwich as ``solve_reduced``.

    This is NOT the reference's preconditioner (which is a single Kronecker
    term, solvers.py:103-196): it changes MO-PCG iteration counts, so it is
    judged on converged-solution parity only.  For a two-term operator it is
    the exact inverse (one iteration)."""

    mode = "two-term-spectral"
    is_identity = False
    left = right = None

    def __init__(self, terms, left_name: str = "two-term", right_name: str = "(lam_i+mu_j)",
                 eig: str = "device"):
        self._op = SylvesterOperator(terms, symmetric=True, positive_definite=True)
        if len(self._op) != 2:
            raise SolverError(f"two-term preconditioner needs two nonzero terms, got {len(self._op)}")
        self.cache = build_spectral_cache(self._op, eig=eig)
        self.cache.check_pencils()
        self.shape = self._op.shape
        self.left_name, self.right_name = left_name, right_name

    def native(self, shape=None):
        if shape is not None and tuple(shape) != self.shape:
            raise OperatorError(f"grid shape {tuple(shape)} does not match preconditioner {self.shape}")
        return self.cache.native()

    def apply(self, U):
        return self._op.apply(U)

    def apply_inverse(self, U):
        on_dev = nat.is_device(U)
        t = nat.torch()
        Ud = nat.to_device(U)
        qy, qx = Ud.shape
        if (qy, qx) != self.shape:
            raise OperatorError(f"grid shape {(qy, qx)} does not match preconditioner {self.shape}")
        Z = t.empty_like(Ud)
        nat.check(nat.lib().sfb_pre_apply(self.native(), nat.ptr(Ud), qx, nat.ptr(Z), qx, nat.stream()),
                  "apply_inverse")
        return Z if on_dev else nat.to_host(Z)


def two_term_preconditioner(op: SylvesterOperator, which=(0, 1), eig: str = "device") -> TwoTermPreconditioner:
    """The two-term spectral preconditioner built from terms ``which`` of an
    operator (reference term order, operators.py:198-204 / 272-278): for the
    general elliptic operator (M1, A) + (B1 + gamma M3, M), for the parabolic
    one (M3 + c B1, M) + (c M1, A); exact for two-term operators.  Its pencils
    are diagonalised on the GPU by default (setup, off the loop)."""
    terms = [op.terms[i] for i in which]
    return TwoTermPreconditioner(terms, eig=eig)


def make_preconditioner(kind: str, x: DirectionSet, y: DirectionSet, *, d_u: float = 1.0,
                        tau: float = 0.0, lumped: bool = False, mode: str | None = None) -> Preconditioner:
    """Named single-term preconditioners (solvers.py:156-196)."""
    if kind == "identity":
        return Preconditioner()
    if kind == "parabolic_lumped":
        kind, lumped = "parabolic", True
    mx, my = x.mats, y.mats
    if lumped and (x.lumped is None or y.lumped is None):
        raise SolverError("lumped preconditioner requested without lumped matrices")
    flat = is_unit_degenerate(y)
    if kind == "elliptic_square":
        return Preconditioner(my.A, mx.A, "A(y)", "A(x)", mode=mode)
    if kind == "elliptic_xnormal":
        if lumped:
            right = mx.A if flat else mx.A + x.lumped.A2
            return Preconditioner(y.lumped.A1, right, "A1(y)", "A(x)" if flat else "A+A2(x)", mode=mode)
        right = mx.A if flat else mx.A + mx.B2
        return Preconditioner(my.B1, right, "B1(y)", "A(x)" if flat else "A+B2(x)", mode=mode)
    if kind == "parabolic":
        c = d_u * tau
        if lumped:
            left = y.lumped.M0 @ y.lumped.D1 + c * y.lumped.A1
            right = x.lumped.M0 + c * (mx.A if flat else mx.A + x.lumped.A2)
            return Preconditioner(left, right, "M0*D1+d*tau*A1(y)", "M0+d*tau*(A+A2)(x)", mode=mode)
        left = my.M3 + c * my.B1
        right = mx.M + c * (mx.A if flat else mx.A + mx.B2)
        return Preconditioner(left, right, "M3+d*tau*B1(y)", "M+d*tau*(A+B2)(x)", mode=mode)
    raise SolverError(f"unknown preconditioner kind '{kind}'")


# ------------------------------------------------------ spectral solve -----
def _fix_eigvectors(vecs):
    """Largest-magnitude entry of each column positive (solvers.py:203-208).
    Device tensors stay on the device."""
    if nat.is_device(vecs):
        t = nat.torch()
        idx = t.argmax(vecs.abs(), dim=0)
        signs = t.sign(vecs[idx, t.arange(vecs.shape[1], device=vecs.device)])
        signs[signs == 0] = 1.0
        return (vecs * signs).contiguous()
    idx = np.argmax(np.abs(vecs), axis=0)
    signs = np.sign(vecs[idx, np.arange(vecs.shape[1])])
    signs[signs == 0] = 1.0
    return vecs * signs


def _min_abs_pair_sum(a: np.ndarray, b: np.ndarray) -> float:
    """min_ij |a_i + b_j| in O(n log n) (b sorted)."""
    bs = np.sort(b)
    pos = np.searchsorted(bs, -a)
    best = np.full(a.shape, np.inf)
    for p in (pos - 1, pos):
        ok = (p >= 0) & (p < bs.size)
        best[ok] = np.minimum(best[ok], np.abs(a[ok] + bs[p[ok]]))
    return float(best.min())


def _host_mat(m) -> np.ndarray:
    return m.cpu().numpy() if nat.is_device(m) else m


@dataclass
class SpectralCache:
    """Eigen-factorisations of the two pencils of a two-term equation
    (solvers.py:211-253); the device sandwich is built on first use.  P1/P2
    are numpy arrays (host eigensolver) or CUDA tensors (device eigensolver:
    they never leave the GPU on the solve path)."""

    lam1: np.ndarray
    lam2: np.ndarray
    P1: np.ndarray
    P2: np.ndarray
    G2: object
    H1: object
    swapped: bool

    @property
    def X1(self):
        return _host_mat(self.P1)

    @property
    def X1inv(self):
        return _host_mat(self.P1).T @ np.asarray(self.G2)

    @property
    def X2(self):
        return np.asarray(self.H1) @ _host_mat(self.P2)

    @property
    def X2inv(self):
        return _host_mat(self.P2).T

    def kernel(self) -> np.ndarray:
        self.check_pencils()
        return 1.0 / (self.lam1[:, None] + self.lam2[None, :])

    def check_pencils(self) -> None:
        if not self.__dict__.get("_pencils_ok"):
            if _min_abs_pair_sum(self.lam1, self.lam2) < PENCIL_GUARD:
                raise SolverError("spectral pencils are (numerically) singular: an eigenvalue "
                                  f"sum fell below {PENCIL_GUARD:g}")
            self._pencils_ok = True

    def reduced(self, op) -> int:
        """Native reduced-solve object of (this cache, op): the sandwich and
        the residual captured into one CUDA graph (sfb_reduced_*)."""
        d = self.__dict__.setdefault("_reduced", {})
        key = id(op)
        e = d.get(key)
        if e is None or e[0]() is not op:
            L = nat.lib()
            out = nat.C.c_void_p()
            nat.check(L.sfb_reduced_create(self.native(), op.native(), nat.C.byref(out)), "reduced solve")
            selfref = weakref.ref(self)

            def _evict(ref, key=key, selfref=selfref):
                c = selfref()
                ent = c.__dict__.get("_reduced", {}).get(key) if c is not None else None
                if ent is not None and ent[0] is ref:
                    del c.__dict__["_reduced"][key]

            # weak in the operator (op._direct_cache -> this cache -> op would be a cycle);
            # the native object keeps the operator's native handle alive itself
            e = (weakref.ref(op, _evict), nat.Handle(out.value, L.sfb_reduced_destroy), op._handle, self._handle)
            d[key] = e
        return e[1].p

    def native(self):
        h = getattr(self, "_handle", None)
        if h is None:
            L = nat.lib()
            qy, qx = self.P1.shape[0], self.P2.shape[0]
            out = nat.C.c_void_p()

            # device tensors are read in place (sfb_pre_create copies device to device)
            keep = [m.contiguous() if nat.is_device(m) else np.ascontiguousarray(m) for m in (self.P1, self.P2)]
            ptrs = [nat.ptr(m) if nat.is_device(m) else nat.host_ptr(m) for m in keep]
            nat.check(L.sfb_pre_create(qy, qx, nat.PRE_SPECTRAL_SUM, ptrs[0], ptrs[1],
                                       nat.host_ptr(np.ascontiguousarray(self.lam1)),
                                       nat.host_ptr(np.ascontiguousarray(self.lam2)), nat.C.byref(out)),
                      "spectral cache")
            h = nat.Handle(out.value, L.sfb_pre_destroy)
            self._handle = h
        return h.p


    def uses_strassen(self) -> int:
        """Strassen levels of the four products of the spectral sandwich (0: one
        DMMA GEMM each; see set_strassen_min_q)."""
        return int(nat.lib().sfb_pre_uses_strassen(self.native()))


def _dense_device(m):
    """Dense fp64 CUDA copy of a factor; band-stored factors are scattered on
    the device from their (row, col, value) triplets (no dense host array)."""
    t = nat.torch()
    if isinstance(m, Band):
        c = m.sparse.tocoo()
        out = t.zeros(m.shape, dtype=t.float64, device="cuda")
        rows = t.from_numpy(c.row.astype(np.int64)).cuda()
        cols = t.from_numpy(c.col.astype(np.int64)).cuda()
        out.index_put_((rows, cols), t.from_numpy(np.asarray(c.data, dtype=float)).cuda(), accumulate=True)
        return out
    return t.from_numpy(np.ascontiguousarray(np.asarray(m, dtype=float))).cuda()


def _geigh_device(A, B):
    """Generalized SPD eigenproblem A v = lam B v on the GPU (setup only),
    through the C ABI (``sfb_geigh``: cuSOLVER potrf + syevd, cuBLAS trsm,
    the reference's sign rule applied on the device).  Eigenvectors are
    B-orthonormal like LAPACK dsygvd's."""
    t = nat.torch()
    Ad, Bd = _dense_device(A), _dense_device(B)
    q = Ad.shape[0]
    lam = np.zeros(q)
    V = t.empty((q, q), dtype=t.float64, device="cuda")
    rc = nat.lib().sfb_geigh(q, nat.ptr(Ad), Ad.stride(0), nat.ptr(Bd), Bd.stride(0), nat.dptr(lam), nat.ptr(V), q,
                             nat.stream())
    if rc == nat.ERR_ARG:
        raise np.linalg.LinAlgError(nat.last_error())
    nat.check(rc, "generalized eigensolver")
    return lam, V


def build_spectral_cache(op: SylvesterOperator, eig: str = "host") -> SpectralCache:
    """Generalized SPD eigh of both pencils with term-order auto-detection
    (solvers.py:256-281).  ``eig="host"`` (default) is LAPACK dsygvd, the
    reference's own route (parity to ~1e-14, SURVEY finding 6);
    ``eig="device"`` is Cholesky + cuSOLVER syevd on the GPU (much faster at
    q >= 4096; ~1e-11 differences for near-singular pencils)."""
    if len(op.terms) != 2:
        raise SolverError(f"spectral reduction needs a two-term operator, got {len(op.terms)} terms")
    if eig not in ("host", "device"):
        raise SolverError(f"unknown eigensolver route '{eig}'")
    geigh = (lambda A, B: sla.eigh(np.asarray(A), np.asarray(B))) if eig == "host" else _geigh_device
    last = None
    for i, j, swapped in ((0, 1, False), (1, 0, True)):
        (G1, H1), (G2, H2) = op.terms[i], op.terms[j]
        try:
            lam1, P1 = geigh(G1, G2)
            lam2, P2 = geigh(H2, H1)
        except (np.linalg.LinAlgError, sla.LinAlgError) as exc:
            last = exc
            continue
        return SpectralCache(lam1=lam1, lam2=lam2, P1=_fix_eigvectors(P1), P2=_fix_eigvectors(P2),
                             G2=G2, H1=H1, swapped=swapped)
    raise SolverError(f"operator is not reducible to Z1 U + U Z2 form: {last}")


def solve_reduced(op: SylvesterOperator, rhs, cache: SpectralCache | None = None) -> SolveReport:
    """U = P1 [(P1^T B P2) / (lam1_i + lam2_j)] P2^T on the device (solvers.py:284-300)."""
    t0 = time.perf_counter()
    if cache is None:
        cache = build_spectral_cache(op)
    cache.check_pencils()
    on_dev = nat.is_device(rhs)
    t = nat.torch()
    B = nat.to_device(rhs)
    qy, qx = B.shape
    if (qy, qx) != tuple(op.shape):
        raise OperatorError(f"grid shape {(qy, qx)} does not match operator {op.shape}")
    U = t.empty_like(B)
    out2 = np.zeros(2)
    nat.check(nat.lib().sfb_reduced_solve(cache.reduced(op), nat.ptr(B), qx, nat.ptr(U), qx, nat.dptr(out2),
                                          nat.stream()), "reduced solve")
    res = out2[0] / max(out2[1], 1e-300)
    return SolveReport(solution=U if on_dev else nat.to_host(U), method="reduced", iterations=0,
                       residual_history=np.array([res]), stop_reason="direct",
                       wall_time=time.perf_counter() - t0,
                       diagnostics={"pencil_swapped": cache.swapped})


def dirichlet_p1_eigenvalues(N: int, gamma: float = 0.0) -> np.ndarray:
    """Closed-form eigenvalues of M^-1 A + gamma/2, P1 Dirichlet (solvers.py:303-312)."""
    i = np.arange(1, N)
    lam_a = 2.0 * N * (1.0 - np.cos(i * np.pi / N))
    return ((12.0 * N * N - gamma) * lam_a + 6.0 * N * gamma) / (12.0 * N - 2.0 * lam_a)


def dirichlet_sine_basis(N: int) -> np.ndarray:
    i = np.arange(1, N)
    return np.sin(np.outer(i, i) * np.pi / N)


def solve_reduced_closed_form(gamma: float, f_nodal, N: int) -> SolveReport:
    """Sine-basis spectral solve, P1 Dirichlet square (solvers.py:321-354).

    With V = sqrt(2/N) X (orthogonal, symmetric) the reference's
    (2/N) X [(1/(lam_i+lam_j)) o ((2/N) X F X)] X is the device sandwich
    V [(V F V) / (lam_i + lam_j)] V."""
    t0 = time.perf_counter()
    on_dev = nat.is_device(f_nodal)
    F = nat.to_device(f_nodal)
    q = N - 1
    if tuple(F.shape) != (q, q):
        raise SolverError(f"closed-form path needs a square {q} x {q} nodal source, got {tuple(F.shape)}")
    if gamma < 0:
        raise SolverError("reaction coefficient must be nonnegative")
    lam = dirichlet_p1_eigenvalues(N, gamma)
    if _min_abs_pair_sum(lam, lam) < PENCIL_GUARD:
        raise SolverError("singular eigenvalue sum in closed-form reduction")
    V = np.ascontiguousarray(np.sqrt(2.0 / N) * dirichlet_sine_basis(N))
    cache = SpectralCache(lam1=lam, lam2=lam, P1=V, P2=V, G2=None, H1=None, swapped=False)
    t = nat.torch()
    L = nat.lib()
    U = t.empty_like(F)
    h = cache.native()
    nat.check(L.sfb_pre_apply(h, nat.ptr(F), q, nat.ptr(U), q, nat.stream()), "closed form")
    fh = t.empty_like(F)
    uh = t.empty_like(F)
    nat.check(L.sfb_pre_transform(h, nat.ptr(F), q, nat.ptr(fh), q, nat.stream()), "transform")
    nat.check(L.sfb_pre_transform(h, nat.ptr(U), q, nat.ptr(uh), q, nat.stream()), "transform")
    lt = t.from_numpy(lam).to("cuda")
    denom = lt[:, None] + lt[None, :]
    res = float(t.linalg.norm(denom * uh - fh) / max(float(t.linalg.norm(fh)), 1e-300))
    return SolveReport(solution=U if on_dev else nat.to_host(U), method="reduced-closed", iterations=0,
                       residual_history=np.array([res]), stop_reason="direct",
                       wall_time=time.perf_counter() - t0,
                       diagnostics={"residual_space": "spectral"})


# --------------------------------------------------------------- MO-PCG ----
_REASONS = {nat.PCG_TOLERANCE: "tolerance", nat.PCG_INCREMENT: "increment", nat.PCG_MAX_ITER: "max_iter"}


class _PcgSolver:
    """Device MO-PCG workspace bound to one (operator, preconditioner) pair.

    It keeps the two native objects it points into (the operator's and the
    preconditioner's handles) alive, but not the Python operator or
    preconditioner: the cache entry lives on the operator, so a reference
    back to it would be a cycle that only the cyclic GC frees."""

    def __init__(self, op: SylvesterOperator, pre):
        L = nat.lib()
        out = nat.C.c_void_p()
        nat.check(L.sfb_pcg_create(op.native(), pre.native(op.shape), nat.C.byref(out)), "mo_pcg")
        self.handle = nat.Handle(out.value, L.sfb_pcg_destroy)
        owner = getattr(pre, "cache", pre)  # TwoTermPreconditioner: the spectral cache owns the sandwich
        self._keep = (op._handle, getattr(owner, "_handle", None))


def _identity_for(op: SylvesterOperator) -> Preconditioner:
    """One identity preconditioner per operator (mo_pcg's precond=None), so
    repeated solves reuse one cached device solver."""
    pre = op.__dict__.get("_identity_pre")
    if pre is None:
        pre = op._identity_pre = Preconditioner()
    return pre


def _solver_for(op: SylvesterOperator, pre) -> _PcgSolver:
    """The cached device solver of (op, pre).  Entries are keyed by the
    preconditioner's identity and dropped when that preconditioner dies (a
    weak reference with an eviction callback), so a loop that builds a fresh
    preconditioner per call does not accumulate device workspaces."""
    key = id(pre)
    cache = op._pcg_cache
    e = cache.get(key)
    if e is not None and e[0]() is pre:
        return e[1]
    solver = _PcgSolver(op, pre)
    opref = weakref.ref(op)

    def _evict(ref, key=key, opref=opref):
        o = opref()
        if o is not None:
            ent = o._pcg_cache.get(key)
            if ent is not None and ent[0] is ref:
                del o._pcg_cache[key]

    cache[key] = (weakref.ref(pre, _evict), solver)
    return solver


def _cached_solver(op: SylvesterOperator, pre):
    e = op._pcg_cache.get(id(pre))
    return e[1] if e is not None and e[0]() is pre else None


def pcg_pass_times(op: SylvesterOperator, precond: Preconditioner | None = None, reps: int = 20) -> dict:
    """Device ms per launch of the passes of one MO-PCG iteration (banded
    operator, vector update, preconditioner) on the solver that `mo_pcg`
    built for (op, precond); call after a solve.  Measurement helper for the
    roofline report (no reference counterpart)."""
    precond = precond if precond is not None else _identity_for(op)
    s = _cached_solver(op, precond)
    if s is None:
        raise SolverError("pcg_pass_times needs a prior mo_pcg solve with this operator and preconditioner")
    ms = np.zeros(3)
    nat.check(nat.lib().sfb_pcg_pass_times(s.handle.p, int(reps), nat.dptr(ms)), "pass timing")
    return {"operator_ms": float(ms[0]), "update_ms": float(ms[1]), "preconditioner_ms": float(ms[2])}


_ITERATES_FIRST = 64  # record_iterates: slots of the first attempt


def mo_pcg(op: SylvesterOperator, rhs, precond: Preconditioner | None = None,
           stop: StoppingRule | None = None, u0=None, max_iter: int = DEFAULT_MAX_ITER,
           record_iterates: bool = False) -> SolveReport:
    """Conjugate gradients with grid-matrix iterates (solvers.py:365-453).

    Numpy in -> numpy out (drop-in); CUDA tensors in -> CUDA tensors out.
    ``diagnostics["dense_grid_matrices"]`` keeps the reference's memory-model
    constant (5); the device workspace is reported under ``"device"``."""
    if not (op.symmetric and op.positive_definite):
        raise OperatorError("mo_pcg needs an operator flagged self-adjoint positive definite")
    if precond is None:
        precond = _identity_for(op)
    if stop is None:
        stop = relative_residual(DEFAULT_TOL)
    t0 = time.perf_counter()
    on_dev = nat.is_device(rhs)
    t = nat.torch()
    B = nat.to_device(rhs)
    qy, qx = op.shape
    if tuple(B.shape) != (qy, qx):
        raise OperatorError(f"grid shape {tuple(B.shape)} does not match operator {op.shape}")
    U0 = None if u0 is None else nat.to_device(u0)
    if U0 is not None and tuple(U0.shape) != (qy, qx):
        raise OperatorError(f"grid shape {tuple(U0.shape)} does not match operator {op.shape}")
    solver = _solver_for(op, precond)
    U = t.empty((qy, qx), dtype=t.float64, device="cuda")
    hist = np.zeros(max_iter + 1)
    incs = np.zeros(max(max_iter, 1))
    rule = stop.native_kind

    def solve(cap):
        its = t.empty((cap, qy, qx), dtype=t.float64, device="cuda") if cap else None
        res = nat.PcgResult()
        nat.check(nat.lib().sfb_pcg_solve(
            solver.handle.p, nat.ptr(B), qx, nat.ptr(U0) if U0 is not None else None, qx, nat.ptr(U), qx,
            rule, float(stop.value), int(max_iter), nat.dptr(hist), nat.dptr(incs),
            nat.ptr(its) if its is not None else None, cap, nat.C.byref(res), nat.stream()), "mo_pcg")
        return res, its

    # record_iterates: the reference appends only the iterates it computes
    # (solvers.py:400, 441-442).  Record into a modest buffer first; a longer
    # solve is re-run with exactly n + 1 slots (every reduction is
    # deterministic, so the second run retraces the first bit for bit).
    cap = min(max_iter + 1, _ITERATES_FIRST) if record_iterates else 0
    res, its = solve(cap)
    n = res.iterations
    if record_iterates and n + 1 > cap:
        del its
        res, its = solve(n + 1)
        n = res.iterations
    if res.stop_reason == nat.PCG_INDEFINITE:
        raise OperatorError("operator is not positive definite along a search direction "
                            f"(<L(Q), Q> = {res.bad_value:.3e} at iteration {res.bad_iter})")
    if res.stop_reason == nat.PCG_NONFINITE:
        raise SolverError(f"mo_pcg residual became non-finite at iteration {res.bad_iter}")
    diag = {"dense_grid_matrices": 5, "increments": incs[:n].copy(),
            "preconditioner": (precond.left_name, precond.right_name)
            if not precond.is_identity else ("identity", "identity"),
            "stopping_rule": stop.describe(),
            "device": {"loop_ms": res.device_ms, "graph_launches": res.chunks,
                       "precond_mode": "identity" if precond.is_identity else precond.mode,
                       "operator": "banded" if op.banded else "dense"}}
    if record_iterates:
        host = nat.to_host(its[: n + 1])
        diag["iterates"] = [host[i] for i in range(n + 1)]
    return SolveReport(solution=U if on_dev else nat.to_host(U), method="mo-pcg", iterations=n,
                       residual_history=hist[: n + 1].copy(), stop_reason=_REASONS[res.stop_reason],
                       wall_time=time.perf_counter() - t0, diagnostics=diag)


# ------------------------------------------- Kronecker cross-check path ----
class _DeviceCSR:
    """A sparse vec-form matrix uploaded once for the device SpMV."""

    def __init__(self, K):
        K = sp.csr_matrix(K)
        K.sort_indices()
        n = K.shape[0]
        if K.shape != (n, n):
            raise OperatorError(f"vector_pcg needs a square matrix, got {K.shape}")
        self.n, self.nnz = n, int(K.nnz)
        indptr = np.ascontiguousarray(K.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(K.indices, dtype=np.int32)
        data = np.ascontiguousarray(K.data, dtype=float)
        L = nat.lib()
        out = nat.C.c_void_p()
        nat.check(L.sfb_csr_create(n, self.nnz, nat.host_ptr(indptr), nat.host_ptr(indices), nat.host_ptr(data),
                                   nat.C.byref(out)), "csr")
        self.handle = nat.Handle(out.value, L.sfb_csr_destroy)

    def matvec(self, x, y):
        nat.check(nat.lib().sfb_csr_spmv(self.handle.p, nat.ptr(x), nat.ptr(y), nat.stream()), "spmv")


class _DeviceLU:
    """A generic sparse preconditioner P factored once on the host like the
    reference (SuperLU: Pr P Pc = L U, solvers.py:473) and solved on the
    device (sfb_lu_solve: permutations and level-scheduled triangular
    sweeps in one kernel)."""

    def __init__(self, P, n: int):
        import scipy.sparse.linalg as spla
        P = sp.csc_matrix(P, dtype=float)
        if P.shape != (n, n):
            raise OperatorError(f"preconditioner of shape {P.shape} does not match the {n} unknowns")
        try:
            f = spla.splu(P)
        except RuntimeError as exc:  # singular factor
            raise SolverError(f"preconditioner factorisation failed: {exc}") from None
        Lc, Uc = sp.csr_matrix(f.L), sp.csr_matrix(f.U)
        arrs = []
        for M in (Lc, Uc):
            M.sort_indices()
            arrs.append((np.ascontiguousarray(M.indptr, dtype=np.int64), np.ascontiguousarray(M.indices, np.int32),
                         np.ascontiguousarray(M.data, dtype=float)))
        # P^-1 r = Pc U^-1 L^-1 Pr r: (Pr r)[perm_r[i]] = r[i], (Pc x)[i] = x[perm_c[i]]
        pr = np.ascontiguousarray(f.perm_r, dtype=np.int32)
        pc = np.ascontiguousarray(f.perm_c, dtype=np.int32)
        L = nat.lib()
        out = nat.C.c_void_p()
        (lp, li, lv), (up, ui, uv) = arrs
        nat.check(L.sfb_lu_create(n, int(lv.size), nat.host_ptr(lp), nat.host_ptr(li), nat.host_ptr(lv), int(uv.size),
                                  nat.host_ptr(up), nat.host_ptr(ui), nat.host_ptr(uv), nat.host_ptr(pr),
                                  nat.host_ptr(pc), nat.C.byref(out)), "sparse LU")
        self.handle = nat.Handle(out.value, L.sfb_lu_destroy)

    def solve(self, r, z):
        nat.check(nat.lib().sfb_lu_solve(self.handle.p, nat.ptr(r), nat.ptr(z), nat.stream()), "sparse LU solve")


def _vec_ops(n):
    """Host-synchronous vector passes (the sharded MO-PCG blocks) on 1 x n rows."""
    L = nat.lib()

    def update(x, r, q, w, alpha):  # x += alpha q; r -= alpha w; -> |r|^2
        out = np.zeros(1)
        nat.check(L.sfb_vec_update(nat.ptr(x), nat.ptr(r), nat.ptr(q), nat.ptr(w), n, 1, n, float(alpha),
                                   nat.dptr(out), nat.stream()), "update")
        return float(out[0])

    def dots(a, b, c=None, d=None):
        out = np.zeros(2)
        nat.check(L.sfb_vec_dots(nat.ptr(a), nat.ptr(b), nat.ptr(c) if c is not None else None,
                                 nat.ptr(d) if d is not None else None, n, 1, n, nat.dptr(out), nat.stream()),
                  "dots")
        return float(out[0]), float(out[1])

    def xpby(q, z, beta, first=False):  # q = z + beta q
        nat.check(L.sfb_vec_xpby(nat.ptr(q), n, nat.ptr(z), n, 1, n, float(beta), int(first), nat.stream()), "xpby")

    return update, dots, xpby


def vector_pcg(K, b, P=None, stop: StoppingRule | None = None, x0=None, max_iter: int = DEFAULT_MAX_ITER,
               record_iterates: bool = False) -> SolveReport:
    """Classical vector PCG on the assembled sparse system (solvers.py:456-517),
    the independent cross-check of mo_pcg, on the device: CSR SpMV kernel,
    fused update / dot / direction passes.  ``P`` is None (identity) or a
    Kronecker-structured preconditioner from ``Preconditioner.as_kronecker``,
    whose inverse runs through the preconditioner's own device kernels
    (the reference factors P with SuperLU)."""
    if stop is None:
        stop = relative_residual(DEFAULT_TOL)
    t0 = time.perf_counter()
    t = nat.torch()
    Kd = _DeviceCSR(K)
    n = Kd.n
    bh = np.asarray(b, dtype=float).reshape(-1)
    if bh.size != n:
        raise OperatorError(f"right-hand side of length {bh.size} does not match the {n} x {n} matrix")
    pre = lu = None
    if P is not None:
        pre = getattr(P, "sfb_pre", None)
        if pre is not None:  # Kronecker-structured: the preconditioner's own device kernels
            qy, qx = P.sfb_shape
            if qy * qx != n:
                raise OperatorError(f"preconditioner of grid {P.sfb_shape} does not match the {n} unknowns")
        else:  # any sparse P: factored once (solvers.py:473), solved on the device
            lu = _DeviceLU(P, n)

    def solve_p(r, z):
        if lu is not None:
            lu.solve(r, z)
            return
        if pre is None:
            z.copy_(r)
            return
        U = r.view(qx, qy).t().contiguous()  # unvec (column stacking)
        Zm = pre.apply_inverse(U)
        z.copy_(Zm.t().contiguous().view(1, n))

    update, dots, xpby = _vec_ops(n)
    dev = lambda a: t.from_numpy(np.ascontiguousarray(a, dtype=float).reshape(1, n)).cuda()  # noqa: E731
    B = dev(bh)
    x = dev(np.zeros(n) if x0 is None else x0)
    r = B.clone()
    w = t.empty_like(B)
    if x0 is not None:
        Kd.matvec(x, w)
        r.sub_(w)  # r = b - K x0 (solvers.py:476)
    res0 = math.sqrt(dots(r, r)[0])
    history = [res0]
    iterates = [nat.to_host(x).reshape(-1)] if record_iterates else None

    def report(iters, reason):
        diag = {"iterates": iterates} if record_iterates else {}
        return SolveReport(solution=nat.to_host(x).reshape(-1), method="vector-pcg", iterations=iters,
                           residual_history=np.asarray(history), stop_reason=reason,
                           wall_time=time.perf_counter() - t0, diagnostics=diag)

    if res0 == 0.0:
        return report(0, "tolerance")
    z = t.empty_like(B)
    q = t.empty_like(B)
    solve_p(r, z)
    xpby(q, z, 0.0, first=True)
    rz = dots(r, z)[0]
    for s in range(max_iter):
        Kd.matvec(q, w)
        qw, qq = dots(q, w, q, q)
        if qw <= 0.0:
            raise OperatorError("matrix is not positive definite along a direction")
        alpha = rz / qw
        res = math.sqrt(update(x, r, q, w, alpha))
        history.append(res)
        if record_iterates:
            iterates.append(nat.to_host(x).reshape(-1))
        if stop.kind == "residual" and res <= stop.value * res0:
            return report(s + 1, "tolerance")
        if stop.kind == "increment" and abs(alpha) * math.sqrt(qq) <= stop.value:
            return report(s + 1, "increment")
        solve_p(r, z)
        rz_new = dots(r, z)[0]
        beta = rz_new / rz
        rz = rz_new
        xpby(q, z, beta)
    return report(max_iter, "max_iter")


def solve_direct(op: SylvesterOperator, rhs) -> SolveReport:
    """Solution of the Kronecker system to round-off (solvers.py:521-555).

    The reference factors to_kronecker(op) with sparse LU.  Here symmetric
    positive definite operators are solved entirely on the device: the
    spectral reduced solve for two-term operators, otherwise MO-PCG to a
    1e-14 relative residual with the two-term spectral preconditioner of the
    operator's first two terms.  Any other operator takes the reference's
    own route — SuperLU factors of the Kronecker matrix (host, once), the
    triangular solves on the device (sfb_lu_solve); an exactly singular
    factor raises SolverError like the reference.  The reference's Kronecker
    guard, relative-residual check (> 1e-9 -> SolverError) and report fields
    are kept."""
    t0 = time.perf_counter()
    rhs = np.asarray(rhs, dtype=float)
    K = to_kronecker(op)  # the reference's guard and the residual check below
    if tuple(rhs.shape) != tuple(op.shape):
        raise OperatorError(f"grid shape {rhs.shape} does not match operator {op.shape}")
    if not (op.symmetric and op.positive_definite):
        t = nat.torch()
        n = K.shape[0]
        lu = _DeviceLU(K, n)
        zd = t.empty((1, n), dtype=t.float64, device="cuda")
        lu.solve(t.from_numpy(np.ascontiguousarray(vec(rhs)).reshape(1, n)).cuda(), zd)
        U = unvec(nat.to_host(zd).reshape(-1), op.shape)
    else:
        try:
            if len(op.terms) == 2:
                U = solve_reduced(op, rhs).solution
            else:
                pre = two_term_preconditioner(op)
                U = mo_pcg(op, rhs, precond=pre, stop=relative_residual(1e-14), max_iter=100000).solution
        except (SolverError, np.linalg.LinAlgError):
            U = mo_pcg(op, rhs, stop=relative_residual(1e-14), max_iter=100000).solution
    b = vec(rhs)
    Kd = _DeviceCSR(K)
    t = nat.torch()
    xd = t.from_numpy(np.ascontiguousarray(vec(U))).cuda()
    yd = t.empty_like(xd)
    Kd.matvec(xd, yd)
    Kx = nat.to_host(yd)
    res = float(np.linalg.norm(Kx - b) / max(np.linalg.norm(b), 1e-300))
    if not np.all(np.isfinite(U)) or res > 1e-9:
        raise SolverError(f"sparse direct solve failed (relative residual {res:.2e}; singular operator?)")
    return SolveReport(solution=np.asarray(U), method="direct", iterations=0, residual_history=np.array([res]),
                       stop_reason="direct", wall_time=time.perf_counter() - t0,
                       diagnostics={"nnz": int(K.nnz), "n": int(K.shape[0])})
