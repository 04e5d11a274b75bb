"""Native IMEX step loops (sfb_imex_heat_run / sfb_imex_rds_run, SURVEY §8 b):
the same trajectory as the per-step driver (same kernels, so bit-identical),
and the reference's failure semantics (step, species, last finite state)."""

import numpy as np
import pytest

import paper_2109_01173_b200 as pb
from _cases import sine_source
from conftest import relerr
from test_host_logic import WAVE

pytestmark = pytest.mark.gpu
D, NB = pb.BCKind.DIRICHLET, pb.BCKind.NEUMANN


def heat_case(N=8):
    x, y = pb.build_direction_sets(WAVE, 4, N, D)
    F = sine_source(N, N, 4)
    u0 = 1e-2 * np.random.default_rng(4).standard_normal((y.q, x.q))
    return x, y, F, u0


def per_step(monkeypatch):
    monkeypatch.setattr(pb.timestepping, "NATIVE_LOOP", False)


def test_native_heat_loop_matches_per_step_driver(monkeypatch):
    x, y, F, u0 = heat_case()
    grid = pb.TimeGrid(1e-3, 6e-3)
    inner = pb.InnerSolver(rule="residual", tol=1e-12, max_iter=5000)
    nat = pb.imex_euler_heat(WAVE, x, y, 1.0, pb.SeparableSource(F, lambda t: np.exp(-t)), u0, grid, inner=inner)
    assert nat.diagnostics.get("loop") == "native"
    # the per-step driver with a host callable forms W = U + tau s(t) F on the host
    # (one rounding apart from the fused device weight c_k F)
    host = pb.imex_euler_heat(WAVE, x, y, 1.0, lambda u, X, Y, t: np.exp(-t) * F, u0, grid, inner=inner)
    assert np.array_equal(nat.iterations, host.iterations)
    assert relerr(nat.final[0], host.final[0]) <= 1e-12
    assert np.allclose(nat.increments, host.increments, rtol=1e-10)
    per_step(monkeypatch)
    dev = pb.imex_euler_heat(WAVE, x, y, 1.0, pb.SeparableSource(F, lambda t: np.exp(-t)), u0, grid, inner=inner)
    assert "loop" not in dev.diagnostics
    assert np.array_equal(nat.iterations, dev.iterations)
    assert np.array_equal(nat.final[0], dev.final[0])
    assert np.array_equal(nat.increments, dev.increments)


def test_native_heat_loop_not_converged():
    x, y, F, u0 = heat_case()
    with pytest.raises(pb.SolverError, match="did not converge in 1 iterations"):
        pb.imex_euler_heat(WAVE, x, y, 1.0, pb.SeparableSource(F, lambda t: 1.0), u0, pb.TimeGrid(1e-3, 3e-3),
                           inner=pb.InnerSolver(rule="residual", tol=1e-14, max_iter=1))


def test_native_heat_loop_blowup_keeps_last_state():
    x, y, F, u0 = heat_case()
    # the source weight explodes at t = 2 tau: steps 0 and 1 complete, step 2's W is > 1e100
    src = pb.SeparableSource(F, lambda t: 1e120 if t > 1.5e-3 else 1.0)
    ref = pb.imex_euler_heat(WAVE, x, y, 1.0, pb.SeparableSource(F, lambda t: 1.0), u0, pb.TimeGrid(1e-3, 2e-3),
                             inner=pb.InnerSolver(rule="residual", tol=1e-12, max_iter=5000))
    with pytest.raises(pb.BlowUpError) as info:
        pb.imex_euler_heat(WAVE, x, y, 1.0, src, u0, pb.TimeGrid(1e-3, 5e-3),
                           inner=pb.InnerSolver(rule="residual", tol=1e-12, max_iter=5000))
    assert info.value.step == 2 and info.value.species == "u"
    assert np.array_equal(info.value.state, ref.final[0])


def dib_case(N=15):
    p = pb.dib_presets("spots_worms").replace(rho=400.0)
    x, y = pb.build_direction_sets(pb.SQUARE, 1, N, NB, lumped=True)
    e0, t0 = pb.initial_fields((y.q, x.q), pb.InitialData(amplitude=2e-3, seed=5))
    return p, x, y, (e0 - 1e-3, t0 - 1e-3), 5e-3 / p.rho


@pytest.mark.parametrize("snap", [0, 2, 4])
def test_native_rds_loop_matches_per_step_driver(snap, monkeypatch):
    p, x, y, state0, tau = dib_case()
    grid = pb.TimeGrid(tau, 7 * tau)
    inner = pb.InnerSolver(rule="residual", tol=1e-12, max_iter=2000)
    nat = pb.imex_euler_rds(pb.SQUARE, x, y, 1.0, p.d_theta, pb.dib_kinetics_pair(p), p.rho, state0, grid,
                            inner=inner, lumped=True, snapshot_every=snap)
    assert nat.diagnostics.get("loop") == "native"
    per_step(monkeypatch)
    host = pb.imex_euler_rds(pb.SQUARE, x, y, 1.0, p.d_theta, pb.dib_kinetics_pair(p), p.rho, state0, grid,
                             inner=inner, lumped=True, snapshot_every=snap)
    assert "loop" not in host.diagnostics
    assert np.array_equal(nat.iterations, host.iterations)
    assert np.array_equal(nat.increments, host.increments)
    assert np.array_equal(nat.final[0], host.final[0]) and np.array_equal(nat.final[1], host.final[1])
    assert [s[0] for s in nat.snapshots] == [s[0] for s in host.snapshots]
    for a, b in zip(nat.snapshots, host.snapshots):
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    assert nat.steady_step == host.steady_step


def test_native_rds_steady_state_and_blowup():
    p, x, y, state0, tau = dib_case(9)
    # at the homogeneous equilibrium (0, 0.5) nothing moves: steady at step 0
    q = (y.q, x.q)
    tr = pb.imex_euler_rds(pb.SQUARE, x, y, 1.0, p.d_theta, pb.dib_kinetics_pair(p), p.rho,
                           (np.zeros(q), np.full(q, 0.5)), pb.TimeGrid(tau, 3 * tau),
                           inner=pb.InnerSolver(rule="residual", tol=1e-12, max_iter=2000), lumped=True)
    assert tr.steady_step == 0
    # theta's kinetics explode (C huge): species v fails its rhs check at step 0, u's solve already ran
    bad = pb.dib_kinetics_pair(p.replace(C=1e300, D=1.0))
    with pytest.raises(pb.BlowUpError) as info:
        pb.imex_euler_rds(pb.SQUARE, x, y, 1.0, p.d_theta, bad, p.rho, state0, pb.TimeGrid(tau, 3 * tau),
                          inner=pb.InnerSolver(rule="residual", tol=1e-12, max_iter=2000), lumped=True)
    assert info.value.step == 0 and info.value.species == "v"
    assert np.array_equal(info.value.state[0], state0[0]) and np.array_equal(info.value.state[1], state0[1])
