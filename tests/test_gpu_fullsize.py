"""Parity at the BASELINE.json sizes (SURVEY §8 c).

cfg1 (q = 256) and cfg2 (q = 1024, the swapped pencil) are full reduced
solves, compared with the oracle's reduced solve on the same seeded source
(<= 1e-10 relative Frobenius).  cfg3-cfg5 are too long for a full CPU
reference solve, so SURVEY §8 c's fixed-budget rule applies: the step-0
system of each (cfg3: the elliptic system, K = 10; cfg4: IMEX step 0, rhs
from u0 and the t = 0 source, warm start u0, K = 3; cfg5: both species'
step-0 systems of imex_euler_rds, K = 2) runs K MO-PCG iterations with the
stop rule disabled on the device (reference preconditioner as dense-inverse
products -- on the Strassen schedule at these sizes -- and as banded SPIKE
solves) and in the oracle; the K-th iterates and
the residual histories must agree to <= 1e-10.  The oracle is the checker
(dense GEMM apply, LU preconditioner), never the measured path.
"""

import numpy as np
import pytest

import oracle as orc
import paper_2109_01173_b200 as pb
from conftest import relerr
from paper_2109_01173_b200 import workloads as wl

pytestmark = pytest.mark.gpu


def test_cfg1_full_reduced_solve_vs_oracle():
    w = wl.cfg1()
    assert w.op.shape == (256, 256)
    rep = pb.solve_reduced(w.op, w.rhs)
    ox, oy = orc.direction_sets(orc.unit_square(), 1, w.N, orc.DIRICHLET)
    terms, orhs = orc.elliptic_terms(ox, oy, 1.0)
    rhs = orhs(wl.sine_source(w.N, w.N, 1))
    assert relerr(w.rhs, rhs) <= 1e-13
    U, res, cache = orc.reduced_solve(terms, rhs)
    assert rep.diagnostics["pencil_swapped"] is bool(cache["swapped"])
    assert relerr(rep.solution, U) <= 1e-10
    assert rep.residual_history[-1] <= 1e-10


def test_cfg2_full_reduced_solve_swapped_pencil_vs_oracle():
    """Neumann P3 on [0,2]x[0,1]: the first pencil ordering fails (its B is
    not positive definite), the reference swaps the terms
    (solvers.py:256-281) and lambda_min + mu_min ~ 5e-13 sits near the
    guard."""
    w = wl.cfg2()
    assert w.op.shape == (1024, 1024)
    rep = pb.solve_reduced(w.op, w.rhs)
    ox, oy = orc.direction_sets(orc.rect_domain(), 3, w.N, orc.NEUMANN)
    terms, orhs = orc.elliptic_terms(ox, oy, 0.5)
    rhs = orhs(wl.cosine_source_rect(w.N, 2))
    assert relerr(w.rhs, rhs) <= 1e-13
    U, res, cache = orc.reduced_solve(terms, rhs)
    assert bool(cache["swapped"]) and rep.diagnostics["pencil_swapped"] is True
    assert relerr(rep.solution, U) <= 1e-10


def _fixed_budget(op, kind, kw, x, y, terms, opre, rhs, u0, K):
    ref = orc.mo_pcg(terms, rhs, opre.inverse, ("residual", 1e-300), u0=u0, max_iter=K)
    assert ref["iterations"] == K
    for mode in ("inverse", "banded"):
        pre = pb.make_preconditioner(kind, x, y, mode=mode, **kw)
        if mode == "inverse":  # the BASELINE sizes of cfg3-cfg5 run the dense products on the Strassen schedule
            assert pre.uses_strassen() == (3 if min(op.shape) >= 4000 else 2)
        rep = pb.mo_pcg(op, rhs, precond=pre, stop=pb.fixed_budget(), u0=u0, max_iter=K)
        assert rep.iterations == K and rep.stop_reason == "max_iter", mode
        assert relerr(rep.solution, ref["solution"]) <= 1e-10, mode
        h = np.asarray(ref["history"])
        assert np.max(np.abs(rep.residual_history - h) / h) <= 1e-10, mode
        del pre
    pb.clear_step_cache()


def test_cfg3_full_size_fixed_budget_vs_oracle():
    w = wl.cfg3()
    assert w.op.shape == (2047, 2047)
    ox, oy = orc.direction_sets(orc.wave_domain(), 2, w.N, orc.DIRICHLET)
    terms, orhs = orc.elliptic_terms(ox, oy, 1.0)
    opre = orc.LUPrecond(*orc.precond_factors("elliptic_xnormal", ox, oy))
    rhs = orhs(wl.sine_source(w.N, w.N, 3))
    assert relerr(w.rhs, rhs) <= 1e-13
    _fixed_budget(w.op, "elliptic_xnormal", {}, w.x, w.y, terms, opre, w.rhs, None, 10)


def test_cfg4_step0_full_size_fixed_budget_vs_oracle():
    w = wl.cfg4()
    ex = w.extra
    assert w.op.shape == (4095, 4095)
    ox, oy = orc.direction_sets(orc.wave_domain(), 4, w.N, orc.DIRICHLET)
    terms, orhs = orc.parabolic_terms(ox, oy, 1.0, ex["tau"])
    opre = orc.LUPrecond(*orc.precond_factors("parabolic", ox, oy, d_u=1.0, tau=ex["tau"]))
    u0 = ex["u0"]
    rhs = orhs(orc.expand_full(u0, ox, oy) + ex["tau"] * ex["source"].F)  # IMEX step 0 (t = 0)
    _fixed_budget(w.op, "parabolic", {"d_u": 1.0, "tau": ex["tau"]}, w.x, w.y, terms, opre, rhs, u0, 3)


def test_cfg5_step0_both_species_full_size_fixed_budget_vs_oracle():
    w = wl.cfg5()
    ex = w.extra
    p, tau = ex["params"], ex["tau"]
    assert w.op.shape == (8192, 8192)
    ox, oy = orc.direction_sets(orc.unit_square(), 1, w.N, orc.NEUMANN, lumped=True)
    eta0, th0 = ex["state0"]
    op_p = orc.dib_params(alpha=p.alpha, gamma_k=p.gamma_k, A1=p.A1, A2=p.A2, B=p.B, C=p.C, D=p.D, k2=p.k2,
                          k3=p.k3, d_theta=p.d_theta, rho=p.rho)
    f, g = orc.dib_rates(eta0, th0, op_p)
    for d, S, rate in ((1.0, eta0, f), (p.d_theta, th0, g)):
        terms, orhs = orc.parabolic_terms(ox, oy, d, tau, True)
        opre = orc.LUPrecond(*orc.precond_factors("parabolic_lumped", ox, oy, d_u=d, tau=tau, lumped=True))
        op, _ = pb.parabolic_operator(w.x, w.y, d, tau, lumped=True)
        rhs = orhs(S + tau * p.rho * rate)  # imex_euler_rds step 0 (timestepping.py:200-209)
        _fixed_budget(op, "parabolic_lumped", {"d_u": d, "tau": tau, "lumped": True}, w.x, w.y, terms, opre,
                      rhs, S, 2)
        del terms, opre, op
