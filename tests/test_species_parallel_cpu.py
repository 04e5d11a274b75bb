"""Species-parallel IMEX for the two-species DIB system (SURVEY §8 e,
"Species"), world size 2 over gloo on CPU: the same trajectory as the
single-process oracle, and the same exception on every rank."""

import os
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as orc
from _species_worker import case, oracle_kinetics, worker
from test_sharded_cpu import free_port


def run(mode, N, steps, blow=""):
    d = tempfile.mkdtemp()
    mp.spawn(worker, args=(2, free_port(), mode, d, N, steps, blow), nprocs=2, join=True)
    return [dict(np.load(os.path.join(d, f"rank{r}.npz"))) for r in range(2)]


def test_species_parallel_matches_oracle_trajectory():
    N, steps = 15, 5
    parts = run("cpu", N, steps)
    p, _, _, state0, tau = case(N)
    ox, oy = orc.direction_sets(orc.unit_square(), 1, N, orc.NEUMANN, lumped=True)
    ref = orc.imex_rds(ox, oy, 1.0, p.d_theta, oracle_kinetics(p), p.rho, state0, tau, steps * tau,
                       rule="residual", tol=1e-12, max_iter=2000, lumped=True, snapshot_every=2)
    for r in parts:  # every rank returns the whole trajectory
        assert str(r["err"]) == ""
        assert np.array_equal(r["iters"], ref["iterations"])
        assert np.array_equal(r["U"], ref["final"][0]) and np.array_equal(r["V"], ref["final"][1])
        assert np.array_equal(r["incs"], ref["increments"])
        assert list(r["snaps"]) == [s[0] for s in ref["snapshots"]]


@pytest.mark.parametrize("species", ["u", "v"])
def test_species_parallel_blowup_raised_on_every_rank(species):
    parts = run("cpu", 7, 3, blow=species)
    p, _, _, state0, _ = case(7)
    for r in parts:
        assert str(r["err"]) == f"blowup 0 {species}"
        assert np.array_equal(r["U"], state0[0]) and np.array_equal(r["V"], state0[1])
