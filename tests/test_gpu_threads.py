"""Reentrancy (SURVEY §8 b "Threading"): the reference's harness calls the
solvers from a ThreadPoolExecutor (harness.py:313-317).  Concurrent solves
from several host threads — on shared and on separate operator objects —
must give exactly the results of the same solves run one after another
(every reduction is deterministic, so bit-identical)."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_2109_01173_b200 as pb
from _cases import sine_source
from test_host_logic import WAVE

pytestmark = pytest.mark.gpu


def problems():
    out = []
    for k, N, mode in ((2, 24, "inverse"), (2, 32, "banded"), (1, 40, "spectral"), (3, 24, "inverse")):
        x, y = pb.build_direction_sets(WAVE, k, N, pb.BCKind.DIRICHLET)
        op, rhs_of = pb.elliptic_operator(x, y, 1.0)
        pre = pb.make_preconditioner("elliptic_xnormal", x, y, mode=mode)
        out.append((op, pre, rhs_of(sine_source(N, N, 3))))
    return out


def solve(args):
    op, pre, rhs = args
    return pb.mo_pcg(op, rhs, precond=pre, stop=pb.relative_residual(1e-12), max_iter=3000)


def test_concurrent_mo_pcg_matches_sequential():
    probs = problems()
    seq = [solve(p) for p in probs]
    work = probs * 3  # the same operator objects shared by several threads
    with ThreadPoolExecutor(max_workers=6) as pool:
        par = list(pool.map(solve, work))
    for i, r in enumerate(par):
        s = seq[i % len(probs)]
        assert r.iterations == s.iterations
        assert np.array_equal(r.solution, s.solution)
        assert np.array_equal(r.residual_history, s.residual_history)


def test_concurrent_reduced_solves_and_imex():
    x, y = pb.build_direction_sets(pb.SQUARE, 1, 33, pb.BCKind.DIRICHLET)
    op, rhs_of = pb.elliptic_operator(x, y, 1.0)
    cache = pb.build_spectral_cache(op)
    rng = np.random.default_rng(5)
    rhss = [rng.standard_normal(op.shape) for _ in range(8)]
    seq = [pb.solve_reduced(op, b, cache).solution for b in rhss]
    with ThreadPoolExecutor(max_workers=4) as pool:
        par = list(pool.map(lambda b: pb.solve_reduced(op, b, cache).solution, rhss))
    for a, b in zip(par, seq):
        assert np.array_equal(a, b)
    p = pb.dib_presets("spots_worms").replace(rho=400.0)
    xn, yn = pb.build_direction_sets(pb.SQUARE, 1, 15, pb.BCKind.NEUMANN, lumped=True)
    e0, t0 = pb.initial_fields((yn.q, xn.q), pb.InitialData(amplitude=2e-3, seed=5))

    def run(_):
        return pb.imex_euler_rds(pb.SQUARE, xn, yn, 1.0, p.d_theta, pb.dib_kinetics_pair(p), p.rho, (e0, t0),
                                 pb.TimeGrid(1.25e-5, 5e-5), lumped=True)
    ref = run(0)
    with ThreadPoolExecutor(max_workers=3) as pool:
        outs = list(pool.map(run, range(3)))
    for tr in outs:
        assert np.array_equal(tr.final[0], ref.final[0]) and np.array_equal(tr.final[1], ref.final[1])
        assert np.array_equal(tr.iterations, ref.iterations)


def test_concurrent_stream_k_gemms_at_full_width():
    """At q >= 1024 every DMMA GEMM is a persistent stream-K grid of one CTA
    per SM (148 CTAs).  Independent solver objects on their own streams, run
    from a thread pool as the reference's harness does (harness.py:313-317),
    launch such grids concurrently; split tiles are finished by their last
    arriving piece, so no CTA waits on a CTA that cannot be scheduled.  Every
    result must equal the sequential one bit for bit."""
    work = []
    for k, N, dom in ((1, 1025, pb.SQUARE), (2, 1040, WAVE), (1, 1100, WAVE)):
        x, y = pb.build_direction_sets(dom, k, N, pb.BCKind.DIRICHLET)
        op, rhs_of = pb.elliptic_operator(x, y, 1.0)
        kind = "elliptic_xnormal" if dom is WAVE else "elliptic_square"
        pre = pb.make_preconditioner(kind, x, y, mode="inverse")
        assert min(op.shape) >= 1024
        work.append(("pcg", op, pre, rhs_of(sine_source(N, N, 4))))
    x, y = pb.build_direction_sets(pb.SQUARE, 1, 1200, pb.BCKind.DIRICHLET)
    opr, rhs_of = pb.elliptic_operator(x, y, 1.0)
    cache = pb.build_spectral_cache(opr)
    rng = np.random.default_rng(11)
    for _ in range(3):
        work.append(("red", opr, cache, rng.standard_normal(opr.shape)))

    def run(item):
        kind, op, aux, rhs = item
        if kind == "pcg":
            rep = pb.mo_pcg(op, rhs, precond=aux, stop=pb.fixed_budget(), max_iter=25)
            return rep.solution, rep.residual_history
        return pb.solve_reduced(op, rhs, aux).solution, None

    seq = [run(w) for w in work]
    for _ in range(3):
        with ThreadPoolExecutor(max_workers=len(work)) as pool:
            par = list(pool.map(run, work * 2))
        for i, (sol, hist) in enumerate(par):
            s_sol, s_hist = seq[i % len(work)]
            assert np.array_equal(sol, s_sol)
            if hist is not None:
                assert np.array_equal(hist, s_hist)
