"""Worker for the world_size > 1 gloo tests of the sharded MO-PCG (CPU).

The collective/halo/transpose logic under test is the product's
(paper_2109_01173_b200.distributed); the local compute is a numpy backend
built from the oracle's dense factors (test infrastructure)."""

import os

import numpy as np
import torch
import torch.distributed as dist

import oracle as orc
from _cases import sine_source
from paper_2109_01173_b200.distributed import Comm, Layout, sharded_mo_pcg


class NumpyBackend:
    def __init__(self, terms, Linv, RinvT, layout, b, banded=False):
        self.L, self.b = layout, b
        self.banded = banded  # the SPIKE route: right solves on row shards, left solves on column shards
        self.terms = terms
        self.Linv, self.RinvT = Linv, RinvT
        qx, n, c0 = layout.qx, layout.n, layout.c0
        self.Hsub = []
        for _, H in terms:
            hs = np.zeros((n + 2 * b, n))
            for e in range(n + 2 * b):
                gcol = c0 - b + e
                if 0 <= gcol < qx:
                    hs[e] = H[gcol, c0:c0 + n]
            self.Hsub.append(hs)

    def zeros(self, r, c):
        return torch.zeros((r, c), dtype=torch.float64)

    def from_host(self, a):
        return torch.from_numpy(np.array(a, dtype=float, copy=True))

    def copy(self, X):
        return X.clone()

    def apply_ext(self, ext, st=None):
        e = ext.numpy()
        return torch.from_numpy(sum(G @ e @ hs for (G, _), hs in zip(self.terms, self.Hsub)))

    def right_T(self, R_rows, st=None):
        return torch.from_numpy(self.RinvT @ R_rows.numpy().T)

    def left(self, XcT, st=None):
        return torch.from_numpy(self.Linv @ XcT.numpy().T)

    def right_rows(self, Xr, st=None):  # Xr P_R^-1
        return torch.from_numpy(Xr.numpy() @ self.RinvT.T)

    def left_cols(self, Xc, st=None):  # P_L^-1 Xc
        return torch.from_numpy(self.Linv @ Xc.numpy())

    def update(self, U, R, Q, W, alpha):
        U += alpha * Q
        R -= alpha * W
        return float((R * R).sum())

    def xpby(self, Q, Z, beta, first=False):
        if first:
            Q.copy_(Z)
        else:
            Q.mul_(beta).add_(Z)

    def dots(self, A, B, C=None, D=None):
        return float((A * B).sum()), (float((C * D).sum()) if C is not None else 0.0)

    def to_host(self, X):
        return X.numpy().copy()

    # -- the device-resident state protocol of sharded_mo_pcg, on the host
    #    (the same arithmetic as the sfb_shard_* kernels) -------------------
    def state(self, max_iter, stop):
        return HostShardState(max_iter, stop)

    def sdots(self, st, A, B, C=None, D=None, slot=0):
        st.slots[slot] = float((A * B).sum())
        if C is not None:
            st.slots[slot + 1] = float((C * D).sum())

    def sstart(self, st):
        st.start()

    def supdate(self, st, U, R, Q, W):
        if st.status != 0:
            return
        wq = float(st.slots[0])
        if not wq > 0.0:
            st.status, st.bad_value, st.bad_iter = 3, wq, st.iter
            return
        st.alpha = st.rz / wq
        st.qq = float(st.slots[1])
        U += st.alpha * Q
        R -= st.alpha * W
        st.slots[2] = float((R * R).sum())

    def scontrol(self, st):
        st.control()

    def sxpby(self, st, Q, Z, first=False):
        if st.status != 0:
            return
        if first:
            Q.copy_(Z)
        else:
            Q.mul_(float(st.slots[4])).add_(Z)

    def sresult(self, st, history=False):
        st.host_reads += 1
        out = (st.status, st.iter, st.bad_iter, st.bad_value)
        if history:
            out += (np.asarray(st.hist), np.asarray(st.incs))
        return out


class HostShardState:
    """Host twin of the sfb_shard_* device state (status codes of the C ABI)."""

    def __init__(self, max_iter, stop):
        self.slots = torch.zeros(8, dtype=torch.float64)
        self.max_iter, self.kind, self.value = max_iter, stop.kind, stop.value
        self.status, self.iter, self.bad_iter, self.bad_value = 0, 0, -1, 0.0
        self.rz = self.alpha = self.qq = self.res0 = 0.0
        self.hist, self.incs, self.host_reads = [], [], 0

    def start(self):
        self.res0 = float(np.sqrt(float(self.slots[2])))
        self.rz = float(self.slots[3])
        self.hist = [self.res0]
        self.status = 1 if self.res0 == 0.0 else (5 if self.max_iter <= 0 else 0)

    def control(self):
        if self.status != 0:
            return
        res = float(np.sqrt(float(self.slots[2])))
        if not np.isfinite(res):
            self.status, self.bad_iter = 4, self.iter
            return
        self.hist.append(res)
        inc = abs(self.alpha) * float(np.sqrt(self.qq))
        self.incs.append(inc)
        self.iter += 1
        if self.kind == "residual" and res <= self.value * self.res0:
            self.status = 1
        elif self.kind == "increment" and inc <= self.value:
            self.status = 2
        elif self.iter >= self.max_iter:
            self.status = 5
        rz_new = float(self.slots[3])
        self.slots[4] = rz_new / self.rz
        self.rz = rz_new


def problem(N, k=2):
    x, y = orc.direction_sets(orc.wave_domain(), k, N, orc.DIRICHLET)
    terms, rhs_of = orc.elliptic_terms(x, y, 1.0)
    L, R, _, _ = orc.precond_factors("elliptic_xnormal", x, y)
    return x, y, terms, rhs_of(sine_source(N, N, 3)), L, R


def worker(rank, world, port, N, out_dir, warm, banded=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, y, terms, rhs, PL, PR = problem(N)
        qy, qx = rhs.shape
        lay = Layout(qy, qx, world, rank)
        b = 2
        be = NumpyBackend(terms, np.linalg.inv(PL), np.linalg.inv(PR).T, lay, b, banded=banded)
        comm = Comm(lay, "cpu")
        # collective unit checks
        rng = np.random.default_rng(7)
        full = rng.standard_normal((qy, qx))
        loc = torch.from_numpy(full[:, lay.c0:lay.c0 + lay.n].copy())
        ext = comm.halo(loc, b).numpy()
        want = np.zeros((qy, lay.n + 2 * b))
        for e in range(lay.n + 2 * b):
            g = lay.c0 - b + e
            if 0 <= g < qx:
                want[:, e] = full[:, g]
        assert np.array_equal(ext, want)
        rows = comm.cols_to_rows(loc).numpy()
        assert np.array_equal(rows, full[lay.r0:lay.r0 + lay.m, :])
        colsT = comm.rowsT_to_colsT(torch.from_numpy(full.T[:, lay.r0:lay.r0 + lay.m].copy())).numpy()
        assert np.array_equal(colsT, full.T[lay.c0:lay.c0 + lay.n, :])
        cols = comm.rows_to_cols(torch.from_numpy(full[lay.r0:lay.r0 + lay.m, :].copy())).numpy()
        assert np.array_equal(cols, full[:, lay.c0:lay.c0 + lay.n])
        u0 = None
        if warm:
            u0 = 1e-2 * np.random.default_rng(4).standard_normal((qy, qx))[:, lay.c0:lay.c0 + lay.n]
        rep = sharded_mo_pcg(be, comm, rhs[:, lay.c0:lay.c0 + lay.n],
                             stop=orc_stop(), u0_local=u0, max_iter=5000)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), U=rep.solution, iters=rep.iterations,
                 hist=rep.residual_history, c0=lay.c0, n=lay.n, host_reads=rep.diagnostics["host_reads"],
                 check_every=rep.diagnostics["check_every"])
    finally:
        dist.destroy_process_group()


def orc_stop():
    from paper_2109_01173_b200.solvers import relative_residual
    return relative_residual(1e-12)
