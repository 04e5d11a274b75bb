"""Sharded MO-PCG with the CUDA backend at world size 2 and 3 (one GPU,
host-staged gloo collectives): same iterations and solution as mo_pcg."""

import os
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2109_01173_b200 as pb
from _sharded_gpu_worker import problem, worker
from conftest import relerr
from test_sharded_cpu import free_port

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_cuda_backend_multirank_matches_mo_pcg(world):
    N = 40
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(worker, args=(world, free_port(), N, d), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    U = np.concatenate([p["U"] for p in parts], axis=1)
    iters = {int(p["iters"]) for p in parts}
    assert len(iters) == 1
    op, pre, rhs = problem(N)
    ref = pb.mo_pcg(op, rhs, precond=pre, stop=pb.relative_residual(1e-12), max_iter=5000)
    # a different GEMM / reduction order per rank count: long solves drift by a
    # couple of iterations (SURVEY finding 6); the solution is the parity check
    assert abs(iters.pop() - ref.iterations) <= max(2, ref.iterations // 200)
    assert relerr(U, ref.solution) <= 1e-10
