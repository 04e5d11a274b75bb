"""GPU tests of the SURVEY §8 f rows (beyond the reference's own algorithm).

f1 (banded preconditioner) is parity-neutral and already runs through every
MO-PCG parity test in tests/test_gpu_parity.py; here: f3, the two-term
spectral preconditioner, which changes iteration counts and is therefore
judged on converged-solution parity against the oracle."""

import numpy as np
import pytest

import oracle as orc
import paper_2109_01173_b200 as pb
from _cases import sine_source, wave_oracle
from conftest import relerr
from test_host_logic import WAVE

pytestmark = pytest.mark.gpu

D, NB = pb.BCKind.DIRICHLET, pb.BCKind.NEUMANN


@pytest.mark.parametrize("N", [16, 48])
def test_two_term_preconditioner_converges_to_reference_solution(N):
    x, y = pb.build_direction_sets(WAVE, 2, N, D)
    op, rhs_of = pb.elliptic_operator(x, y, 1.0)
    rhs = rhs_of(sine_source(N, N, 3))
    pre2 = pb.two_term_preconditioner(op)
    rep2 = pb.mo_pcg(op, rhs, precond=pre2, stop=pb.relative_residual(1e-12), max_iter=5000)
    pre1 = pb.make_preconditioner("elliptic_xnormal", x, y)
    rep1 = pb.mo_pcg(op, rhs, precond=pre1, stop=pb.relative_residual(1e-12), max_iter=5000)
    # oracle: the reference's own (single-term LU) MO-PCG at the same tolerance
    ox, oy = orc.direction_sets(orc.wave_domain(), 2, N, orc.DIRICHLET)
    terms, _ = orc.elliptic_terms(ox, oy, 1.0)
    opre = orc.LUPrecond(*orc.precond_factors("elliptic_xnormal", ox, oy))
    ref = orc.mo_pcg(terms, rhs, opre.inverse, ("residual", 1e-12), max_iter=5000)
    assert rep2.stop_reason == "tolerance"
    assert relerr(rep2.solution, ref["solution"]) <= 1e-10
    # the point of f3: far fewer iterations, independent of N
    assert rep2.iterations < rep1.iterations / 4
    assert rep2.diagnostics["device"]["precond_mode"] == "two-term-spectral"


def test_two_term_preconditioner_is_exact_for_two_term_operators():
    # cfg5-type lumped parabolic operator on the square has exactly two terms
    x, y = pb.build_direction_sets(pb.SQUARE, 1, 31, NB, lumped=True)
    op, _ = pb.parabolic_operator(x, y, 20.0, 5e-3 / 400, lumped=True)
    assert len(op) == 2
    rhs = np.random.default_rng(3).standard_normal(op.shape)
    rep = pb.mo_pcg(op, rhs, precond=pb.two_term_preconditioner(op), stop=pb.relative_residual(1e-12),
                    max_iter=50)
    assert rep.iterations <= 2
    assert relerr(rep.solution, pb.solve_reduced(op, rhs).solution) <= 1e-10


def test_two_term_preconditioner_in_imex_dib():
    p = pb.dib_presets("spots_worms").replace(rho=400.0)
    x, y = pb.build_direction_sets(pb.SQUARE, 1, 15, NB, lumped=True)
    e0, t0 = pb.initial_fields((y.q, x.q), pb.InitialData(amplitude=2e-3, seed=5))
    state0 = (e0 - 1e-3, t0 - 1e-3)
    tau = 5e-3 / p.rho
    grid = pb.TimeGrid(tau, 6 * tau)
    kin = pb.dib_kinetics_pair(p)
    ref = pb.imex_euler_rds(pb.SQUARE, x, y, 1.0, p.d_theta, kin, p.rho, state0, grid, lumped=True,
                            inner=pb.InnerSolver(rule="residual", tol=1e-12, max_iter=2000))
    two = pb.imex_euler_rds(pb.SQUARE, x, y, 1.0, p.d_theta, kin, p.rho, state0, grid, lumped=True,
                            inner=pb.InnerSolver(rule="residual", tol=1e-12, max_iter=2000, precond="two_term"))
    assert np.all(two.iterations <= 2)
    assert relerr(two.final[0], ref.final[0]) <= 1e-10
    assert relerr(two.final[1], ref.final[1]) <= 1e-10


def test_device_eigensolver_route_for_reduced_solves(golden):
    from _cases import cosine_source_rect
    from test_host_logic import RECT
    x, y = pb.build_direction_sets(pb.SQUARE, 1, 17, D)
    op, rhs_of = pb.elliptic_operator(x, y, 1.0)
    c = pb.build_spectral_cache(op, eig="device")
    assert relerr(pb.solve_reduced(op, rhs_of(sine_source(17, 17, 1)), c).solution, golden["red1/U"]) <= 1e-10
    x, y = pb.build_direction_sets(RECT, 3, 12, NB)
    op, rhs_of = pb.elliptic_operator(x, y, 0.5)
    c = pb.build_spectral_cache(op, eig="device")
    assert c.swapped
    assert relerr(pb.solve_reduced(op, rhs_of(cosine_source_rect(12, 2)), c).solution, golden["red2/U"]) <= 1e-10


# f1: the SPIKE banded solves across several 64-row segments, including a
# last segment shorter than the half-bandwidth (q = 64 m + 1, 64 m + 3).
@pytest.mark.parametrize("deg,N,lumped", [(1, 130, False), (2, 130, False), (2, 66, False), (3, 201, False),
                                          (4, 260, False), (1, 200, True)])
def test_banded_preconditioner_multi_segment(deg, N, lumped):
    x, y = pb.build_direction_sets(WAVE, deg, N, D, lumped=lumped)
    kw = dict(lumped=True) if lumped else {}
    pre_b = pb.make_preconditioner("elliptic_xnormal", x, y, mode="banded", **kw)
    pre_i = pb.make_preconditioner("elliptic_xnormal", x, y, mode="inverse", **kw)
    U = np.random.default_rng(deg * 1000 + N).standard_normal((y.q, x.q))
    assert y.q > 64 and x.q > 64
    assert relerr(pre_b.apply_inverse(U), pre_i.apply_inverse(U)) <= 1e-11
    # round trip limited by the factors' conditioning (P4 ~ 1e7), like the LU path
    assert relerr(pre_b.apply(pre_b.apply_inverse(U)), U) <= 1e-8


def test_banded_mode_mo_pcg_multi_segment_vs_oracle():
    """q = 129 (P2): three 64-row SPIKE segments (the last one row long) and
    two banded-kernel strips.
    Both device preconditioner forms against the oracle: iteration counts
    within the oracle's own rounding envelope (+1), solutions <= 1e-10."""
    N = 130
    x, y = pb.build_direction_sets(WAVE, 2, N, D)
    op, rhs_of = pb.elliptic_operator(x, y, 1.0)
    rhs = rhs_of(sine_source(N, N, 3))
    assert op.shape == (129, 129)
    terms, orhs, pinv = wave_oracle(2, N)
    assert relerr(rhs, orhs) <= 1e-13
    ref = orc.mo_pcg(terms, orhs, pinv, ("residual", 1e-12), max_iter=20000)
    it, lo, hi = orc.iteration_envelope(terms, orhs, pinv, ("residual", 1e-12), max_iter=20000)
    assert it == ref["iterations"]
    for m in ("inverse", "banded"):
        rep = pb.mo_pcg(op, rhs, precond=pb.make_preconditioner("elliptic_xnormal", x, y, mode=m),
                        stop=pb.relative_residual(1e-12), max_iter=20000)
        assert abs(rep.iterations - it) <= hi - lo + 1, (m, rep.iterations, it, lo, hi)
        assert relerr(rep.solution, ref["solution"]) <= 1e-10, m


def test_two_term_preconditioner_in_imex_heat_matches_reference_trajectory(golden):
    # cfg4-type (P4, wave domain): the f3 preconditioner changes iteration
    # counts only; at tol 1e-12 the trajectory is the reference's
    x, y = pb.build_direction_sets(WAVE, 4, 8, D)
    F = sine_source(8, 8, 4)
    tr = pb.imex_euler_heat(WAVE, x, y, 1.0, pb.SeparableSource(F, lambda t: np.exp(-t)), golden["heat/u0"],
                            pb.TimeGrid(1e-3, 5e-3),
                            inner=pb.InnerSolver(rule="residual", tol=1e-12, max_iter=5000, precond="two_term"))
    assert np.all(tr.iterations < golden["heat/t12/iters"])
    assert relerr(tr.final[0], golden["heat/t12/U"]) <= 1e-10
    assert np.allclose(tr.increments, golden["heat/t12/incs"], rtol=1e-8)


@pytest.mark.gpu
def test_native_generalized_eigensolver_matches_lapack():
    """sfb_geigh (spectral setup on the device) against scipy.linalg.eigh(A, B)
    (the reference's dsygvd route) with the reference's sign rule."""
    import scipy.linalg as sla

    from paper_2109_01173_b200.solvers import _geigh_device
    rng = np.random.default_rng(9)
    for q in (5, 64, 301):
        X = rng.standard_normal((q, q))
        A = X @ X.T + q * np.eye(q)
        Y = rng.standard_normal((q, q))
        B = Y @ Y.T + q * np.eye(q)
        lam, V = _geigh_device(A, B)
        V = V.cpu().numpy()
        lr, Vr = sla.eigh(A, B)
        idx = np.argmax(np.abs(Vr), axis=0)
        Vr = Vr * np.sign(Vr[idx, np.arange(q)])
        assert np.allclose(lam, lr, rtol=1e-12, atol=0)
        assert np.abs(V - Vr).max() <= 1e-10 * np.abs(Vr).max()
        assert np.allclose(V.T @ B @ V, np.eye(q), atol=1e-10)
        assert np.all(V[np.argmax(np.abs(V), axis=0), np.arange(q)] > 0)
    with pytest.raises(np.linalg.LinAlgError, match="not positive definite"):
        _geigh_device(np.eye(4), -np.eye(4))
