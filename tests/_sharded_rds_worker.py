"""Worker for the column-sharded DIB IMEX tests (gloo).

The halo exchange, the reduced blow-up / norm decisions and the sharded
MO-PCG under test are the product's (distributed.sharded_imex_rds).  On CPU
the local compute is an oracle-built numpy stepper (test infrastructure); on
the GPU it is the product's CudaShardedDibStepper with host-staged
collectives."""

import os

import numpy as np
import torch
import torch.distributed as dist

import oracle as orc
import paper_2109_01173_b200 as pb
from _sharded_worker import NumpyBackend
from _species_worker import case, oracle_kinetics
from paper_2109_01173_b200.distributed import Comm, Layout, grouped_imex_rds, sharded_imex_rds


class OracleShardedDib:
    def __init__(self, N, p, tau, layout, b=1):
        ox, oy = orc.direction_sets(orc.unit_square(), 1, N, orc.NEUMANN, lumped=True)
        self.L, self.b = layout, b
        self.kin = oracle_kinetics(p)
        self.tau_rho = tau * p.rho
        self.backends = []
        for d in (1.0, p.d_theta):
            terms, _ = orc.parabolic_terms(ox, oy, d, tau, True)
            PL, PR, _, _ = orc.precond_factors("parabolic_lumped", ox, oy, d_u=d, tau=tau, lumped=True)
            self.backends.append(NumpyBackend(terms, np.linalg.inv(PL), np.linalg.inv(PR).T, layout, 1))
        ly, d1, ml = orc.mofem._lumped_rows(oy)
        self.G, Hf = ml, ox["lumped"]["M0"]
        q, n, c0 = layout.qx, layout.n, layout.c0
        self.Hsub = np.zeros((n + 2 * b, n))
        for e in range(n + 2 * b):
            g = c0 - b + e
            if 0 <= g < q:
                self.Hsub[e] = Hf[c0:c0 + n, g]

    def to_local(self, a):
        L = self.L
        return torch.from_numpy(np.array(a, dtype=float)[:, L.c0:L.c0 + L.n].copy())

    def rhs(self, sp, extU, extV):
        u, v = extU.numpy(), extV.numpy()
        W = (u if sp == 0 else v) + self.tau_rho * np.asarray(self.kin[sp](u, v))
        fin = np.isfinite(W)
        chk = (float(np.max(np.abs(W[fin]))) if fin.any() else 0.0, float((~fin).sum()))
        return torch.from_numpy(self.G @ W @ self.Hsub), chk

    def norms(self, A, B):
        a, b = A.numpy(), B.numpy()
        return [float(((a - b) ** 2).sum()), float(np.max(np.abs(a))), float((~np.isfinite(a)).sum()),
                float((a * a).sum())]

    def host(self, X):
        return X.numpy().copy()


def worker(rank, world, port, mode, out_dir, N, steps, lumped=True):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, x, y, state0, tau = case(N, lumped)
        lay = Layout(y.q, x.q, world, rank)
        inner = pb.InnerSolver(rule="residual", tol=1e-12, max_iter=2000)
        if mode == "cpu":
            comm, st, kin = Comm(lay, "cpu"), OracleShardedDib(N, p, tau, lay), None
        else:
            from _sharded_gpu_worker import HostStagedComm
            torch.cuda.set_device(0)
            comm, st, kin = HostStagedComm(lay), None, pb.dib_kinetics_pair(p)
        tr = sharded_imex_rds(pb.SQUARE, x, y, 1.0, p.d_theta, kin, p.rho, state0, pb.TimeGrid(tau, steps * tau),
                              inner=inner, lumped=lumped, snapshot_every=2, comm=comm, stepper=st)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), U=tr.final[0], V=tr.final[1], iters=tr.iterations,
                 incs=tr.increments, snaps=[s[0] for s in tr.snapshots], c0=lay.c0)
    finally:
        dist.destroy_process_group()


def grouped_worker(rank, world, port, mode, out_dir, N, steps):
    """Species groups x column shards (world = 2G)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, x, y, state0, tau = case(N)
        inner = pb.InnerSolver(rule="residual", tol=1e-12, max_iter=2000)
        if mode == "cpu":
            kw = dict(device="cpu", stepper_factory=lambda L, g: OracleShardedDib(N, p, tau, L))
            kin = None
        else:
            from _sharded_gpu_worker import HostStagedComm
            torch.cuda.set_device(0)
            kw = dict(device="cpu", comm_factory=lambda L, grp, ranks: HostStagedComm(L, grp, ranks))
            kin = pb.dib_kinetics_pair(p)
        tr = grouped_imex_rds(pb.SQUARE, x, y, 1.0, p.d_theta, kin, p.rho, state0, pb.TimeGrid(tau, steps * tau),
                              inner=inner, lumped=True, snapshot_every=2, **kw)
        if mode != "cpu":
            # a second call reuses the cached per-rank setup (block operators,
            # inverses, species groups) and must retrace the first bit for bit
            tr2 = grouped_imex_rds(pb.SQUARE, x, y, 1.0, p.d_theta, kin, p.rho, state0,
                                   pb.TimeGrid(tau, steps * tau), inner=inner, lumped=True, snapshot_every=2, **kw)
            assert np.array_equal(tr2.final[0], tr.final[0]) and np.array_equal(tr2.final[1], tr.final[1])
            assert np.array_equal(tr2.iterations, tr.iterations)
        c0, c1 = tr.diagnostics["columns"]
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), U=tr.final[0], V=tr.final[1], iters=tr.iterations,
                 incs=tr.increments, snaps=[s[0] for s in tr.snapshots], c0=c0, group=tr.diagnostics["species_group"],
                 snapU=tr.snapshots[0][1], snapV=tr.snapshots[0][2])
    finally:
        dist.destroy_process_group()
