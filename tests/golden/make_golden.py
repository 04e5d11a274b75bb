"""Generate the golden vectors that pin the oracle (and the CUDA path).

Runs the UNMODIFIED reference package (``sylfem`` under
/root/reference/pkg/src, imported read-only) on small seeded instances of the
five BASELINE.json configurations plus assembly/operator cases, and writes
``tests/golden/golden.npz``.  Only this build container has /root/reference;
the GPU box and CI use the committed .npz.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import sylfem as sf  # noqa: E402
from sylfem.geometry import DomainKind, DomainSpec, ProfileFn  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")

D, NB = sf.BCKind.DIRICHLET, sf.BCKind.NEUMANN

WAVE = DomainSpec(DomainKind.XNORMAL, ProfileFn(
    lambda s: 1.0 + 0.3 * np.sin(2 * np.pi * np.asarray(s, float)),
    lambda s: 0.6 * np.pi * np.cos(2 * np.pi * np.asarray(s, float)), name="wave"), name="wave")
RECT = DomainSpec(DomainKind.XNORMAL, ProfileFn(
    lambda s: 2.0 * np.ones_like(np.asarray(s, float)),
    lambda s: np.zeros_like(np.asarray(s, float)), name="rect2"), name="rect")
DOMS = {"square": sf.SQUARE, "cap": sf.CAP_DOMAIN, "jar": sf.JAR_DOMAIN,
        "wave": WAVE, "rect": RECT}
BCS = {"d": D, "n": NB}


def modes(seed):
    rng = np.random.default_rng(seed)
    a = rng.integers(1, 17, 8)
    b = rng.integers(1, 17, 8)
    c = rng.standard_normal(8)
    return a, b, c


def sine_source(N_x, N_y, seed):
    a, b, c = modes(seed)
    xs = np.arange(N_x + 1) / N_x
    ys = np.arange(N_y + 1) / N_y
    return sum(c[m] * np.sin(b[m] * np.pi * ys)[:, None] * np.sin(a[m] * np.pi * xs)[None, :]
               for m in range(8))


def cosine_source_rect(N, seed):
    a, b, c = modes(seed)
    X = 2.0 * np.arange(N + 1) / N
    Y = np.arange(N + 1) / N
    return sum(c[m] * np.cos(b[m] * np.pi * Y)[:, None] * np.cos(a[m] * np.pi * X / 2)[None, :]
               for m in range(8))


def desk_cases():
    """(k, N, domain, bc) of the reference's desk matrix (tests/conftest.py:12-22)."""
    out = []
    for k in (1, 2, 3, 4):
        for n in (8, 16, 24):
            if n % k:
                continue
            for name in ("square", "cap", "jar"):
                for bc in ("d", "n"):
                    out.append((k, n, name, bc))
    return out


def main():
    g = {}
    rng = np.random.default_rng(20260)

    # -- assembly (fem1d.py:246-349) --------------------------------------
    asm_cases = [(1, 8, "square", "d"), (2, 8, "cap", "n"), (3, 12, "jar", "d"),
                 (4, 8, "wave", "d"), (3, 12, "rect", "n"), (2, 10, "wave", "n")]
    for k, n, dn, bc in asm_cases:
        x, y = sf.build_direction_sets(DOMS[dn], k, n, BCS[bc], lumped=(k == 1))
        tag = f"asm/{k}_{n}_{dn}_{bc}"
        for side, s in (("x", x), ("y", y)):
            for name, m in s.mats.named().items():
                g[f"{tag}/{side}/{name}"] = m
            if s.lumped is not None:
                for name, m in s.lumped.named().items():
                    g[f"{tag}/{side}/L_{name}"] = m
    for dn, bc in (("cap", "n"), ("square", "d"), ("jar", "n")):
        x, y = sf.build_direction_sets(DOMS[dn], 1, (9, 6), BCS[bc], lumped=True)
        tag = f"asml/{dn}_{bc}"
        for side, s in (("x", x), ("y", y)):
            for name, m in s.lumped.named().items():
                g[f"{tag}/{side}/{name}"] = m

    # -- operator apply and rhs (operators.py:124-131, 177-284) -----------
    op_cases = [("ell", 1, 8, "square", "d", 0.0, False), ("ell", 2, 8, "cap", "d", 0.0, False),
                ("ell", 3, 12, "jar", "n", 1.0, False), ("ell", 2, 10, "wave", "d", 1.0, False),
                ("ell", 1, 8, "cap", "n", 1.0, True), ("ell", 1, 8, "jar", "d", 0.0, True),
                ("ell", 3, 12, "rect", "n", 0.5, False),
                ("par", 4, 8, "wave", "d", 1e-3, False), ("par", 1, 9, "square", "n", 0.05, True),
                ("par", 2, 8, "cap", "n", 0.01, False)]
    for i, (kind, k, n, dn, bc, p, lumped) in enumerate(op_cases):
        x, y = sf.build_direction_sets(DOMS[dn], k, n, BCS[bc], lumped=lumped)
        if kind == "ell":
            op, rhs_of = sf.elliptic_operator(x, y, p, lumped=lumped)
        else:
            op, rhs_of = sf.parabolic_operator(x, y, 1.0, p, lumped=lumped)
        U = rng.standard_normal(op.shape)
        F = rng.standard_normal((y.basis.n_sub + 1, x.basis.n_sub + 1))
        tag = f"op/{i}"
        g[f"{tag}/U"], g[f"{tag}/AU"] = U, op.apply(U)
        g[f"{tag}/F"], g[f"{tag}/rhs"] = F, rhs_of(F)
        g[f"{tag}/nterms"] = np.array(len(op.terms))

    # -- reduced solves: cfg1-type and cfg2-type (solvers.py:256-300) -----
    x, y = sf.build_direction_sets(sf.SQUARE, 1, 17, D)
    op, rhs_of = sf.elliptic_operator(x, y, 1.0)
    rhs = rhs_of(sine_source(17, 17, 1))
    rep = sf.solve_reduced(op, rhs)
    g["red1/rhs"], g["red1/U"] = rhs, rep.solution
    g["red1/res"], g["red1/swapped"] = rep.residual_history, np.array(rep.diagnostics["pencil_swapped"])
    x, y = sf.build_direction_sets(RECT, 3, 12, NB)
    op, rhs_of = sf.elliptic_operator(x, y, 0.5)
    rhs = rhs_of(cosine_source_rect(12, 2))
    rep = sf.solve_reduced(op, rhs)
    g["red2/rhs"], g["red2/U"] = rhs, rep.solution
    g["red2/res"], g["red2/swapped"] = rep.residual_history, np.array(rep.diagnostics["pencil_swapped"])
    g["red2/nterms"] = np.array(len(op.terms))

    # -- MO-PCG: cfg3-type (solvers.py:365-453) ----------------------------
    x, y = sf.build_direction_sets(WAVE, 2, 16, D)
    op, rhs_of = sf.elliptic_operator(x, y, 1.0)
    pre = sf.make_preconditioner("elliptic_xnormal", x, y)
    rhs = rhs_of(sine_source(16, 16, 3))
    for tol_tag, tol in (("t12", 1e-12), ("t8", 1e-8)):
        rep = sf.mo_pcg(op, rhs, precond=pre, stop=sf.relative_residual(tol),
                        max_iter=5000, record_iterates=True)
        tag = f"pcg3/{tol_tag}"
        g[f"{tag}/U"] = rep.solution
        g[f"{tag}/iters"] = np.array(rep.iterations)
        g[f"{tag}/hist"] = rep.residual_history
        g[f"{tag}/incs"] = rep.diagnostics["increments"]
        g[f"{tag}/first8"] = np.stack(rep.diagnostics["iterates"][:8])
    g["pcg3/rhs"] = rhs
    g["pcg3/names"] = np.array(list(rep.diagnostics["preconditioner"]))
    # preconditioner inverse on a random grid (solvers.py:134-143)
    R = rng.standard_normal(op.shape)
    g["pcg3/R"], g["pcg3/PinvR"] = R, pre.apply_inverse(R)

    # -- IMEX heat: cfg4-type (timestepping.py:126-159) --------------------
    x, y = sf.build_direction_sets(WAVE, 4, 8, D)
    F = sine_source(8, 8, 4)
    src = lambda u, X, Y, t: np.exp(-t) * F
    u0 = 1e-2 * np.random.default_rng(4).standard_normal((y.q, x.q))
    grid = sf.TimeGrid(1e-3, 5e-3)
    g["heat/u0"], g["heat/F"] = u0, F
    for tol_tag, tol in (("t12", 1e-12), ("t8", 1e-8)):
        tr = sf.imex_euler_heat(WAVE, x, y, 1.0, src, u0, grid,
                                inner=sf.InnerSolver(rule="residual", tol=tol, max_iter=5000))
        g[f"heat/{tol_tag}/U"] = tr.final[0]
        g[f"heat/{tol_tag}/iters"] = tr.iterations
        g[f"heat/{tol_tag}/incs"] = tr.increments

    # -- IMEX DIB: cfg5-type (timestepping.py:162-220, models.py:74-126) ---
    p = sf.dib_presets("spots_worms").replace(rho=400.0)
    x, y = sf.build_direction_sets(sf.SQUARE, 1, 15, NB, lumped=True)
    e0, t0 = sf.initial_fields((y.q, x.q), sf.InitialData(amplitude=2e-3, seed=5))
    state0 = (e0 - 1e-3, t0 - 1e-3)
    kin = (lambda u, v: sf.dib_kinetics(u, v, p)[0], lambda u, v: sf.dib_kinetics(u, v, p)[1])
    tau = 5e-3 / p.rho
    g["dib/eta0"], g["dib/theta0"] = state0
    g["dib/D"] = np.array(p.D)
    for tag, inner in (("tau", sf.InnerSolver()), ("t12", sf.InnerSolver(rule="residual", tol=1e-12,
                                                                          max_iter=2000))):
        tr = sf.imex_euler_rds(sf.SQUARE, x, y, 1.0, p.d_theta, kin, p.rho, state0,
                               sf.TimeGrid(tau, 6 * tau), inner=inner, lumped=True,
                               snapshot_every=2)
        g[f"dib/{tag}/U"], g[f"dib/{tag}/V"] = tr.final
        g[f"dib/{tag}/iters"] = tr.iterations
        g[f"dib/{tag}/incs"] = tr.increments
        g[f"dib/{tag}/snap_steps"] = np.array([s[0] for s in tr.snapshots])
    ee = rng.standard_normal((5, 7)) * 0.3
    tt = 0.5 + 0.2 * rng.standard_normal((5, 7))
    fv, gv = sf.dib_kinetics(ee, tt, p)
    g["kin/eta"], g["kin/theta"], g["kin/f"], g["kin/g"] = ee, tt, fv, gv
    g["init/eta"], g["init/theta"] = sf.initial_fields((6, 5), sf.InitialData(amplitude=1e-3, seed=7))

    # -- closed-form reduced solve, k = 1 Dirichlet square (solvers.py:303-354)
    for gamma in (0.0, 1.0):
        n = 16
        x, y = sf.build_direction_sets(sf.SQUARE, 1, n, D)
        F = sine_source(n, n, 6)
        rep = sf.solve_reduced_closed_form(gamma, sf.interior_values(F, x, y), n)
        tag = f"closed/g{int(gamma)}"
        g[f"{tag}/F"], g[f"{tag}/U"] = F, rep.solution
        g[f"{tag}/res"] = rep.residual_history

    # -- the acceptance desk matrix (tests/test_acceptance.py:109-154 with
    #    tests/conftest.py:12-30): per case a random apply, the direct
    #    solution, the reduced and closed-form solutions where they apply and
    #    the MO-PCG solve (reference preconditioner for Dirichlet, identity
    #    for Neumann) ---------------------------------------------------------
    for i, (k, n, name, bc) in enumerate(desk_cases()):
        drng = np.random.default_rng(1234 + i)
        bck = BCS[bc]
        x, y = sf.build_direction_sets(sf.domain_from_name(name), k, n, bck, lumped=k == 1)
        gamma = 0.0 if bck is D else 1.0
        op, rhs_of = sf.elliptic_operator(x, y, gamma)
        tag = f"desk/{i}"
        U = drng.standard_normal(op.shape)
        F = drng.standard_normal((y.basis.n_sub + 1, x.basis.n_sub + 1))
        rhs = rhs_of(F)
        g[f"{tag}/U"], g[f"{tag}/AU"] = U, op.apply(U)
        g[f"{tag}/F"], g[f"{tag}/rhs"] = F, rhs
        g[f"{tag}/nterms"] = np.array(len(op.terms))
        g[f"{tag}/direct"] = sf.solve_direct(op, rhs).solution
        if len(op.terms) == 2:
            g[f"{tag}/reduced"] = sf.solve_reduced(op, rhs).solution
            if k == 1 and bck is D and name == "square":
                F0 = F.copy()
                F0[0, :] = F0[-1, :] = F0[:, 0] = F0[:, -1] = 0.0
                g[f"{tag}/reduced0"] = sf.solve_reduced(op, rhs_of(F0)).solution
                g[f"{tag}/closed"] = sf.solve_reduced_closed_form(gamma, sf.interior_values(F0, x, y), n).solution
        if bck is D:
            pre = sf.make_preconditioner("elliptic_square" if name == "square" else "elliptic_xnormal", x, y)
        else:
            pre = sf.make_preconditioner("identity", x, y)
        rep = sf.mo_pcg(op, rhs, precond=pre, stop=sf.relative_residual(1e-12), max_iter=5000)
        g[f"{tag}/pcg"], g[f"{tag}/pcg_iters"] = rep.solution, np.array(rep.iterations)

    np.savez_compressed(OUT, **g)
    print(f"wrote {len(g)} arrays to {OUT} ({os.path.getsize(OUT) / 1024:.0f} KiB)")


if __name__ == "__main__":
    main()
