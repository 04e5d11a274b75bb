"""Worker for the multi-rank test of the CUDA backend of the sharded MO-PCG.

Every rank computes with the product's CudaBackend (C ABI kernels) on the one
visible GPU; the collectives go through gloo on host copies (HostStagedComm),
so the ranks only meet on the host and no kernel waits on another rank's.
This checks the backend's multi-rank logic (halo-extended block operator,
transposed GEMM shards, device dots) — not NVLink performance."""

import os

import numpy as np
import torch
import torch.distributed as dist

import paper_2109_01173_b200 as pb
from _cases import sine_source
from paper_2109_01173_b200.distributed import Comm, CudaBackend, Layout, PeerTransposes, sharded_mo_pcg
from test_host_logic import WAVE


class HostStagedComm:
    """Comm interface of distributed.sharded_mo_pcg over gloo: CUDA tensors
    are staged through host memory for each collective."""

    def __init__(self, layout, group=None, ranks=None):
        self.L = layout
        self.inner = Comm(layout, "cpu", group=group, ranks=ranks)

    def allreduce(self, vals):
        return self.inner.allreduce(vals)

    def allreduce_(self, t):
        h = t.cpu()
        self.inner.allreduce_(h)
        t.copy_(h)
        return t

    def halo_(self, Xe, n, b):
        h = Xe.cpu()
        self.inner.halo_(h, n, b)
        Xe.copy_(h)
        return Xe

    def halo(self, X, b):
        return self.inner.halo(X.cpu(), b).to(X.device)

    def cols_to_rows(self, Xc):
        return self.inner.cols_to_rows(Xc.cpu()).to(Xc.device)

    def rows_to_cols(self, Xr):
        return self.inner.rows_to_cols(Xr.cpu()).to(Xr.device)

    def rowsT_to_colsT(self, XrT):
        return self.inner.rowsT_to_colsT(XrT.cpu()).to(XrT.device)

    def sendrecv(self, X, peer):
        return self.inner.sendrecv(X.cpu(), peer).to(X.device)

    def gather_world(self, vals):
        return self.inner.gather_world(vals)


def problem(N, mode="inverse"):
    x, y = pb.build_direction_sets(WAVE, 2, N, pb.BCKind.DIRICHLET)
    op, rhs_of = pb.elliptic_operator(x, y, 1.0)
    pre = pb.make_preconditioner("elliptic_xnormal", x, y, mode=mode)
    return op, pre, rhs_of(sine_source(N, N, 3))


def worker(rank, world, port, N, out_dir, peer=False, mode="inverse"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        op, pre, rhs = problem(N, mode)
        qy, qx = rhs.shape
        lay = Layout(qy, qx, world, rank)
        be = CudaBackend(op, pre, lay)
        comm = HostStagedComm(lay)
        # peer: the transposes over CUDA IPC mappings (P2P copies + the scatter GEMM),
        # synchronised on the host so ranks sharing the GPU never wait on each other's kernels
        pt = PeerTransposes(lay, be, sync="host") if peer else None
        rep = sharded_mo_pcg(be, comm, rhs[:, lay.c0:lay.c0 + lay.n], stop=pb.relative_residual(1e-12),
                             max_iter=5000, peer=pt)
        if pt is not None:
            torch.cuda.synchronize()
            dist.barrier()
            pt.close()
        from paper_2109_01173_b200 import _native as nat
        levels = [nat.lib().sfb_const_levels(h.p) for h in getattr(be, "_const", {}).values()]
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), U=rep.solution, iters=rep.iterations,
                 hist=rep.residual_history, strassen_levels=min(levels) if levels else 0)
    finally:
        dist.destroy_process_group()


def heat_case(N=24, k=4):
    """cfg4-type: heat on the wave domain, P_k, Dirichlet, separable source."""
    x, y = pb.build_direction_sets(WAVE, k, N, pb.BCKind.DIRICHLET)
    F = sine_source(N, N, 4)
    u0 = 1e-2 * np.random.default_rng(4).standard_normal((y.q, x.q))
    src = pb.SeparableSource(F, lambda t: float(np.exp(-t)))
    inner = pb.InnerSolver(rule="residual", tol=1e-12, max_iter=5000)
    return x, y, src, u0, pb.TimeGrid(1e-3, 4e-3), inner


def heat_worker(rank, world, port, N, out_dir, mode="inverse"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2109_01173_b200.distributed import sharded_imex_heat
        torch.cuda.set_device(0)
        x, y, src, u0, grid, inner = heat_case(N)
        inner = pb.InnerSolver(rule="residual", tol=1e-12, max_iter=5000, precond_mode=mode)
        lay = Layout(y.q, x.q, world, rank)
        tr = sharded_imex_heat(WAVE, x, y, 1.0, src, u0, grid, inner=inner, comm=HostStagedComm(lay))
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), U=tr.final[0], iters=tr.iterations,
                 incs=tr.increments)
    finally:
        dist.destroy_process_group()
