"""Column-sharded MO-PCG (SURVEY §8 e) on CPU with gloo, world_size 2 and 3.

Checks the product's halo exchange, all-to-all transposes and the sharded
recurrences against the single-process oracle MO-PCG on the same system."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as orc
from _sharded_worker import problem, worker
from conftest import relerr


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,warm,banded", [(2, False, False), (3, True, False), (3, False, True)])
def test_sharded_mo_pcg_matches_single_process(world, warm, banded):
    """banded: the SPIKE form's route (right solves on row shards, rows -> cols
    all-to-all, left solves on column shards)."""
    N = 24
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(worker, args=(world, free_port(), N, d, warm, banded), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
        U = np.concatenate([p["U"] for p in parts], axis=1)
        iters = {int(p["iters"]) for p in parts}
    assert len(iters) == 1
    x, y, terms, rhs, PL, PR = problem(N)
    pre = orc.LUPrecond(PL, PR)
    u0 = 1e-2 * np.random.default_rng(4).standard_normal(rhs.shape) if warm else None
    ref = orc.mo_pcg(terms, rhs, pre.inverse, ("residual", 1e-12), u0=u0, max_iter=5000)
    it = iters.pop()
    assert abs(it - ref["iterations"]) <= 1
    assert relerr(U, ref["solution"]) <= 1e-10
    # device-resident loop: the host reads the state once per chunk of
    # iterations (+ setup and the final report), never per iteration
    for p in parts:
        assert int(p["host_reads"]) <= -(-it // int(p["check_every"])) + 6  # + the 1, 2, 4, 8 ramp
