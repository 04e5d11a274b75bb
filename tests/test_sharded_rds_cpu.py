"""Column-sharded DIB IMEX (SURVEY §8 e, cfg5's sharding) at world size 2 and
3 over gloo on CPU, against the single-process oracle trajectory."""

import os
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as orc
from _sharded_rds_worker import grouped_worker, worker
from _species_worker import case, oracle_kinetics
from conftest import relerr
from test_sharded_cpu import free_port


def gather(d, world):
    parts = [dict(np.load(os.path.join(d, f"rank{r}.npz"))) for r in range(world)]
    U = np.concatenate([p["U"] for p in parts], axis=1)
    V = np.concatenate([p["V"] for p in parts], axis=1)
    return parts, U, V


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_rds_matches_oracle_trajectory(world):
    N, steps = 15, 4
    d = tempfile.mkdtemp()
    mp.spawn(worker, args=(world, free_port(), "cpu", d, N, steps), nprocs=world, join=True)
    parts, U, V = gather(d, world)
    p, _, _, state0, tau = case(N)
    ox, oy = orc.direction_sets(orc.unit_square(), 1, N, orc.NEUMANN, lumped=True)
    ref = orc.imex_rds(ox, oy, 1.0, p.d_theta, oracle_kinetics(p), p.rho, state0, tau, steps * tau,
                       rule="residual", tol=1e-12, max_iter=2000, lumped=True, snapshot_every=2)
    for r in parts:
        assert np.all(np.abs(r["iters"] - ref["iterations"]) <= 1)
        assert np.allclose(r["incs"], ref["increments"], rtol=1e-8)
        assert list(r["snaps"]) == [s[0] for s in ref["snapshots"]]
    assert relerr(U, ref["final"][0]) <= 1e-10
    assert relerr(V, ref["final"][1]) <= 1e-10


@pytest.mark.parametrize("world", [2, 4])
def test_grouped_species_sharded_rds_matches_oracle(world):
    """cfg5's 4/8-GPU layout: species groups of world/2 column shards each."""
    N, steps = 15, 4
    d = tempfile.mkdtemp()
    mp.spawn(grouped_worker, args=(world, free_port(), "cpu", d, N, steps), nprocs=world, join=True)
    parts = [dict(np.load(os.path.join(d, f"rank{r}.npz"))) for r in range(world)]
    G = world // 2
    p, _, _, state0, tau = case(N)
    ox, oy = orc.direction_sets(orc.unit_square(), 1, N, orc.NEUMANN, lumped=True)
    ref = orc.imex_rds(ox, oy, 1.0, p.d_theta, oracle_kinetics(p), p.rho, state0, tau, steps * tau,
                       rule="residual", tol=1e-12, max_iter=2000, lumped=True, snapshot_every=2)
    for r in parts:
        assert np.all(np.abs(r["iters"] - ref["iterations"]) <= 1)
        assert np.allclose(r["incs"], ref["increments"], rtol=1e-8)
        assert list(r["snaps"]) == [s[0] for s in ref["snapshots"]]
    for grp in (0, 1):  # each group's ranks return both species on their columns
        mine = sorted((r for r in parts if int(r["group"]) == grp), key=lambda r: int(r["c0"]))
        U = np.concatenate([r["U"] for r in mine], axis=1)
        V = np.concatenate([r["V"] for r in mine], axis=1)
        assert relerr(U, ref["final"][0]) <= 1e-10 and relerr(V, ref["final"][1]) <= 1e-10
        sU = np.concatenate([r["snapU"] for r in mine], axis=1)
        assert relerr(sU, ref["snapshots"][0][1]) <= 1e-10
