"""Sharded MO-PCG with the CUDA backend at world size 2 and 3 (one GPU,
host-staged gloo collectives): same iterations and solution as mo_pcg."""

import os
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as orc
import paper_2109_01173_b200 as pb
from _cases import wave_oracle
from _sharded_gpu_worker import worker
from conftest import relerr
from test_host_logic import WAVE
from test_sharded_cpu import free_port

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,peer,mode", [(2, False, "inverse"), (3, False, "inverse"), (2, True, "inverse"),
                                             (3, True, "inverse"), (2, False, "banded"), (3, True, "banded")])
def test_sharded_cuda_backend_multirank_matches_mo_pcg(world, peer, mode):
    """mode banded: SPIKE solves on the shards (right factor on row shards,
    left factor on column shards) with the rows -> cols exchange."""
    N = 40
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(worker, args=(world, free_port(), N, d, peer, mode), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    U = np.concatenate([p["U"] for p in parts], axis=1)
    iters = {int(p["iters"]) for p in parts}
    assert len(iters) == 1
    # a different GEMM / reduction order per rank count changes the rounding:
    # the iteration count must stay inside the reference's own rounding
    # envelope (the oracle under a deliberate rounding change, +1)
    terms, rhs, pinv = wave_oracle(2, N)
    ref = orc.mo_pcg(terms, rhs, pinv, ("residual", 1e-12), max_iter=5000)
    it, lo, hi = orc.iteration_envelope(terms, rhs, pinv, ("residual", 1e-12), max_iter=5000)
    assert abs(iters.pop() - it) <= hi - lo + 1
    assert relerr(U, ref["solution"]) <= 1e-10


@pytest.mark.parametrize("world,peer", [(2, True), (3, False)])
def test_sharded_cuda_backend_multirank_strassen_products(world, peer, monkeypatch):
    """The shards' products with the full P_L^-1 / P_R^-T as prepared constant operands on the
    Strassen schedule (threshold lowered through the environment of the spawned ranks; q = 95 is
    odd: padded inside the passes), incl. the assembly pass that scatters to the peers' buffers."""
    monkeypatch.setenv("SYLFEM_B200_STRASSEN_MINQ", "64")
    N = 96
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(worker, args=(world, free_port(), N, d, peer, "inverse"), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    assert all(int(p["strassen_levels"]) >= 1 for p in parts)
    U = np.concatenate([p["U"] for p in parts], axis=1)
    iters = {int(p["iters"]) for p in parts}
    assert len(iters) == 1
    terms, rhs, pinv = wave_oracle(2, N)
    ref = orc.mo_pcg(terms, rhs, pinv, ("residual", 1e-12), max_iter=5000)
    it, lo, hi = orc.iteration_envelope(terms, rhs, pinv, ("residual", 1e-12), max_iter=5000)
    assert abs(iters.pop() - it) <= hi - lo + 1
    assert relerr(U, ref["solution"]) <= 1e-10


def test_constant_operand_products_match_the_plain_gemm():
    """sfb_shard_gemm_const / sfb_shard_gemm_scatter_const (prepared constant left operand, Strassen
    schedule) against the plain product and the scatter layout."""
    import torch

    from paper_2109_01173_b200 import _native as nat
    from paper_2109_01173_b200.distributed import Layout, ShardState

    L = nat.lib()
    rng = np.random.default_rng(4)
    qx, m, world, off = 302, 77, 3, 5
    A = torch.from_numpy(rng.standard_normal((qx, qx))).cuda()
    B = torch.from_numpy(rng.standard_normal((m, qx))).cuda()
    ref = (A @ B.T).cpu().numpy()
    prev = pb.set_strassen_min_q(64)
    try:
        out = nat.C.c_void_p()
        nat.check(L.sfb_const_create(A.data_ptr(), qx, qx, qx, m, nat.C.byref(out)), "const")
        const = nat.Handle(out.value, L.sfb_const_destroy)
    finally:
        pb.set_strassen_min_q(prev)
    assert L.sfb_const_levels(const.p) == 2  # leaves of 76 x 76 (left) and 20 x 76 (right)
    st = ShardState(10, pb.fixed_budget())
    C = torch.zeros((qx, m + (m % 2)), dtype=torch.float64, device="cuda")
    nat.check(L.sfb_shard_gemm_const(st.handle.p, const.p, B.data_ptr(), qx, m, C.data_ptr(), C.stride(0), nat.stream()),
              "gemm")
    assert relerr(C[:, :m].cpu().numpy(), ref) <= 1e-13
    lay = Layout(qy=150, qx=qx, world=world, rank=0)
    bufs = [torch.full((lay.col_counts[s], 130 + 2 * s), np.nan, dtype=torch.float64, device="cuda")
            for s in range(world)]
    seg = (nat.C.c_int * (world + 1))(*(list(lay.col_offs) + [qx]))
    dst = (nat.C.c_void_p * world)(*[b.data_ptr() for b in bufs])
    ldd = (nat.C.c_int * world)(*[b.stride(0) for b in bufs])
    nat.check(L.sfb_shard_gemm_scatter_const(st.handle.p, const.p, B.data_ptr(), qx, m, world, seg, dst, ldd, off,
                                             nat.stream()), "scatter")
    torch.cuda.synchronize()
    for s_ in range(world):
        got = bufs[s_].cpu().numpy()
        want = ref[lay.col_offs[s_]:lay.col_offs[s_] + lay.col_counts[s_]]
        assert relerr(got[:, off:off + m], want) <= 1e-13
        assert np.isnan(got[:, :off]).all() and np.isnan(got[:, off + m:]).all()  # nothing else touched
    # a thinner right operand than prepared for, and one too wide (falls back to the plain GEMM)
    nat.check(L.sfb_shard_gemm_const(st.handle.p, const.p, B.data_ptr(), qx, 40, C.data_ptr(), C.stride(0), nat.stream()),
              "gemm")
    assert relerr(C[:, :40].cpu().numpy(), ref[:, :40]) <= 1e-13


def test_scatter_gemm_places_rows_like_the_transpose():
    """sfb_dgemm_nt_scatter with three local destinations (stand-ins for the
    ranks' column-shard buffers) against the plain GEMM and the layout."""
    import torch

    from paper_2109_01173_b200 import _native as nat
    from paper_2109_01173_b200.distributed import Layout

    rng = np.random.default_rng(3)
    qx, m, world, off = 302, 77, 3, 5  # even leading dimensions (TMA rows)
    A = torch.from_numpy(rng.standard_normal((qx, qx))).cuda()
    B = torch.from_numpy(rng.standard_normal((m, qx))).cuda()
    ref = (A @ B.T).cpu().numpy()
    lay = Layout(qy=150, qx=qx, world=world, rank=0)
    bufs = [torch.full((lay.col_counts[s], 130 + 2 * s), np.nan, dtype=torch.float64, device="cuda")
            for s in range(world)]
    seg = (nat.C.c_int * (world + 1))(*(list(lay.col_offs) + [qx]))
    dst = (nat.C.c_void_p * world)(*[b.data_ptr() for b in bufs])
    ldd = (nat.C.c_int * world)(*[b.stride(0) for b in bufs])
    nat.check(nat.lib().sfb_dgemm_nt_scatter(A.data_ptr(), qx, B.data_ptr(), qx, qx, m, qx, world, seg, dst, ldd,
                                              off, nat.stream()), "scatter")
    for s in range(world):
        got = bufs[s].cpu().numpy()
        c0, n = lay.col_offs[s], lay.col_counts[s]
        assert np.allclose(got[:, off:off + m], ref[c0:c0 + n, :], rtol=1e-13, atol=1e-12)
        assert np.all(np.isnan(got[:, :off])) and np.all(np.isnan(got[:, off + m:]))  # nothing outside the block


@pytest.mark.parametrize("world,mode", [(2, "inverse"), (3, "banded")])
def test_sharded_imex_heat_matches_single_gpu_driver(world, mode):
    """cfg4-type heat (P4, wave domain, Dirichlet) with U column-sharded:
    block rhs map over the halo-extended block (fused heat loader), the
    sharded MO-PCG per step; against imex_euler_heat on one GPU."""
    from _sharded_gpu_worker import heat_case, heat_worker
    N = 24
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(heat_worker, args=(world, free_port(), N, d, mode), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
        U = np.concatenate([p["U"] for p in parts], axis=1)
        iters = parts[0]["iters"]
        incs = parts[0]["incs"]
    x, y, src, u0, grid, inner = heat_case(N)
    inner = pb.InnerSolver(rule="residual", tol=1e-12, max_iter=5000, precond_mode=mode)
    ref = pb.imex_euler_heat(WAVE, x, y, 1.0, src, u0, grid, inner=inner)
    assert np.all(np.abs(iters - ref.iterations) <= 2)
    assert relerr(U, ref.final[0]) <= 1e-10
    assert np.allclose(incs, ref.increments, rtol=1e-8)


def test_sharded_imex_heat_single_rank_nccl_peer_graph():
    """World 1 over NCCL with the peer-memory transposes (stream sync) and
    CUDA-graph chunks: the configuration bench.py uses on one GPU per rank."""
    import socket

    import torch.distributed as dist

    from _sharded_gpu_worker import heat_case
    from paper_2109_01173_b200.distributed import sharded_imex_heat
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        x, y, src, u0, grid, inner = heat_case(24)
        tr = sharded_imex_heat(WAVE, x, y, 1.0, src, u0, grid, inner=inner, peer_sync="stream", graph=True)
        ref = pb.imex_euler_heat(WAVE, x, y, 1.0, src, u0, grid, inner=inner)
        assert np.all(np.abs(tr.iterations - ref.iterations) <= 2)
        assert relerr(tr.final[0], ref.final[0]) <= 1e-10
    finally:
        dist.destroy_process_group()
