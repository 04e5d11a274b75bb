"""Species-parallel DIB stepping with the CUDA stepper at world size 2 on one
GPU (state exchange staged through host memory over gloo): bit-identical to
the single-GPU imex_euler_rds, and within the reference tolerance of the
golden reference trajectory."""

import os
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2109_01173_b200 as pb
from _species_worker import case, worker
from conftest import relerr
from test_sharded_cpu import free_port

pytestmark = pytest.mark.gpu


def test_species_parallel_cuda_matches_single_gpu_driver():
    N, steps = 15, 6
    d = tempfile.mkdtemp()
    mp.spawn(worker, args=(2, free_port(), "cuda", d, N, steps, ""), nprocs=2, join=True)
    parts = [dict(np.load(os.path.join(d, f"rank{r}.npz"))) for r in range(2)]
    p, x, y, state0, tau = case(N)
    ref = pb.imex_euler_rds(pb.SQUARE, x, y, 1.0, p.d_theta, pb.dib_kinetics_pair(p), p.rho, state0,
                            pb.TimeGrid(tau, steps * tau),
                            inner=pb.InnerSolver(rule="residual", tol=1e-12, max_iter=2000), lumped=True,
                            snapshot_every=2)
    for r in parts:
        assert str(r["err"]) == ""
        assert np.array_equal(r["iters"], ref.iterations)
        assert np.array_equal(r["U"], ref.final[0]) and np.array_equal(r["V"], ref.final[1])
        assert np.array_equal(r["incs"], ref.increments)
        assert list(r["snaps"]) == [s[0] for s in ref.snapshots]
    assert relerr(parts[0]["V"], ref.final[1]) == 0.0


@pytest.mark.parametrize("world,lumped", [(2, True), (3, True), (3, False)])
def test_sharded_rds_cuda_matches_single_gpu_driver(world, lumped):
    """lumped=False: the consistent mass makes the block rhs map read a 1-column halo."""
    from _sharded_rds_worker import worker as sharded_worker
    N, steps = 15, 4
    d = tempfile.mkdtemp()
    mp.spawn(sharded_worker, args=(world, free_port(), "cuda", d, N, steps, lumped), nprocs=world, join=True)
    parts = [dict(np.load(os.path.join(d, f"rank{r}.npz"))) for r in range(world)]
    U = np.concatenate([p["U"] for p in parts], axis=1)
    V = np.concatenate([p["V"] for p in parts], axis=1)
    p, x, y, state0, tau = case(N, lumped)
    ref = pb.imex_euler_rds(pb.SQUARE, x, y, 1.0, p.d_theta, pb.dib_kinetics_pair(p), p.rho, state0,
                            pb.TimeGrid(tau, steps * tau),
                            inner=pb.InnerSolver(rule="residual", tol=1e-12, max_iter=2000), lumped=lumped,
                            snapshot_every=2)
    for r in parts:
        assert np.all(np.abs(r["iters"] - ref.iterations) <= 1)
        assert np.allclose(r["incs"], ref.increments, rtol=1e-8)
        assert list(r["snaps"]) == [s[0] for s in ref.snapshots]
    assert relerr(U, ref.final[0]) <= 1e-10
    assert relerr(V, ref.final[1]) <= 1e-10


@pytest.mark.parametrize("world", [2, 4])
def test_grouped_species_sharded_cuda_matches_single_gpu_driver(world):
    from _sharded_rds_worker import grouped_worker
    N, steps = 15, 4
    d = tempfile.mkdtemp()
    mp.spawn(grouped_worker, args=(world, free_port(), "cuda", d, N, steps), nprocs=world, join=True)
    parts = [dict(np.load(os.path.join(d, f"rank{r}.npz"))) for r in range(world)]
    p, x, y, state0, tau = case(N)
    ref = pb.imex_euler_rds(pb.SQUARE, x, y, 1.0, p.d_theta, pb.dib_kinetics_pair(p), p.rho, state0,
                            pb.TimeGrid(tau, steps * tau),
                            inner=pb.InnerSolver(rule="residual", tol=1e-12, max_iter=2000), lumped=True,
                            snapshot_every=2)
    for r in parts:
        assert np.all(np.abs(r["iters"] - ref.iterations) <= 1)
        assert np.allclose(r["incs"], ref.increments, rtol=1e-8)
    for grp in (0, 1):
        mine = sorted((r for r in parts if int(r["group"]) == grp), key=lambda r: int(r["c0"]))
        U = np.concatenate([r["U"] for r in mine], axis=1)
        V = np.concatenate([r["V"] for r in mine], axis=1)
        assert relerr(U, ref.final[0]) <= 1e-10 and relerr(V, ref.final[1]) <= 1e-10
