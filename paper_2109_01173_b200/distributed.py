"""Column-sharded MO-PCG across the GPUs of one node (SURVEY §8 e).

Each rank owns a contiguous block of grid columns (x direction) of U, R, Z,
Q and W.  Per iteration (the reference recurrences, solvers.py:423-452):

* W = L(Q): left factors act within columns (local); right factors couple
  columns j-b..j+b, so each rank first receives a b-column halo from both
  neighbours (point-to-point) and runs the banded kernel on its extended
  block (``sfb_op_create_block``);
* <W,Q>, |Q|^2 -> one allreduce of 2 doubles -> alpha;
* U += alpha Q, R -= alpha W (local), |R|^2 local;
* Z = P_L^-1 R P_R^-1 with the inverse-form preconditioner: R is transposed
  to row shards by an all-to-all, each rank computes X^T = P_R^-T R_rows^T
  (DMMA GEMM), a second all-to-all returns X^T in column shards and
  Z = P_L^-1 X (DMMA GEMM) is local;
* {|R|^2, <Z,R>} -> one allreduce (computing Z before the stop test is
  result-identical: the residual is unchanged) -> stop test, beta;
* Q = Z + beta Q (local).

So two scalar allreduces, one halo exchange and two all-to-alls per
iteration.  The collectives are ``torch.distributed`` (NCCL over NVLink on
GPUs, gloo in the CPU tests); the local compute is a ``Backend`` — the CUDA
one below (C ABI), or a numpy one in the tests.

The iteration is device-resident: alpha, beta, the residual history and the
stop test live in a device state (``sfb_shard_*``), the scalar all-reduces
run in place on device slots (NCCL on the stream), and every kernel that
changes the iterate is gated on the device status.  The host issues
``check_every`` iterations back to back and reads the status once per
chunk, so no iteration waits on the host; iterations issued after the stop
are no-ops and the result is the per-iteration loop's.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .exceptions import ConfigError, OperatorError, SolverError
from .solvers import SolveReport, StoppingRule, relative_residual


def partition(n: int, parts: int):
    counts = [n // parts + (1 if r < n % parts else 0) for r in range(parts)]
    offs = [0]
    for c in counts[:-1]:
        offs.append(offs[-1] + c)
    return counts, offs


@dataclass
class Layout:
    qy: int
    qx: int
    world: int
    rank: int

    def __post_init__(self):
        self.col_counts, self.col_offs = partition(self.qx, self.world)
        self.row_counts, self.row_offs = partition(self.qy, self.world)

    @property
    def n(self):
        return self.col_counts[self.rank]

    @property
    def c0(self):
        return self.col_offs[self.rank]

    @property
    def m(self):
        return self.row_counts[self.rank]

    @property
    def r0(self):
        return self.row_offs[self.rank]


class Comm:
    """Collectives of the sharded iteration over torch.distributed."""

    def __init__(self, layout: Layout, device, group=None, ranks=None):
        """``ranks``: the global ranks of ``group`` in group order (point-to-point
        peers are addressed by global rank); default: the default group."""
        import torch
        import torch.distributed as dist
        self.t, self.dist = torch, dist
        self.L = layout
        self.device = device
        self.group = group
        self.ranks = list(ranks) if ranks is not None else list(range(layout.world))

    def allreduce(self, vals):
        t = self.t.tensor(vals, dtype=self.t.float64, device=self.device)
        if self.L.world > 1:
            self.dist.all_reduce(t, group=self.group)
        return [float(v) for v in t.tolist()]

    def allreduce_(self, t):
        """In-place sum over the group of a (device) tensor, stream-ordered:
        no host synchronisation with NCCL."""
        if self.L.world > 1:
            self.dist.all_reduce(t, group=self.group)
        return t

    def halo_(self, Xe, n: int, b: int):
        """Fill the b-column halos of the extended block Xe = [left | X | right]
        (q_y x (n + 2b)) from the neighbours, in place (zero at the domain ends)."""
        L = self.L
        if b == 0 or L.world == 1:
            return Xe
        if n < b:
            raise SolverError(f"column shard of {n} columns is narrower than the halo {b}")
        t = self.t
        ops, recv = [], []
        left, right = L.rank - 1, L.rank + 1
        if left >= 0:
            r = t.empty((Xe.shape[0], b), dtype=Xe.dtype, device=Xe.device)
            ops.append(self.dist.P2POp(self.dist.isend, Xe[:, b:2 * b].contiguous(), self.ranks[left],
                                       group=self.group))
            ops.append(self.dist.P2POp(self.dist.irecv, r, self.ranks[left], group=self.group))
            recv.append((slice(0, b), r))
        if right < L.world:
            r = t.empty((Xe.shape[0], b), dtype=Xe.dtype, device=Xe.device)
            ops.append(self.dist.P2POp(self.dist.isend, Xe[:, n:n + b].contiguous(), self.ranks[right],
                                       group=self.group))
            ops.append(self.dist.P2POp(self.dist.irecv, r, self.ranks[right], group=self.group))
            recv.append((slice(n + b, n + 2 * b), r))
        for req in self.dist.batch_isend_irecv(ops):
            req.wait()  # NCCL: the current stream waits, the host does not
        for sl, r in recv:
            Xe[:, sl] = r
        return Xe

    def sendrecv(self, X, peer: int):
        """Swap X with the rank ``peer`` (global rank, default group)."""
        recv = self.t.empty_like(X)
        ops = [self.dist.P2POp(self.dist.isend, X.contiguous(), peer),
               self.dist.P2POp(self.dist.irecv, recv, peer)]
        for req in self.dist.batch_isend_irecv(ops):
            req.wait()
        return recv

    def gather_world(self, vals):
        """All-gather of a few scalars per rank over the default group."""
        t = self.t.tensor(vals, dtype=self.t.float64, device=self.device)
        out = [self.t.empty_like(t) for _ in range(self.dist.get_world_size())]
        self.dist.all_gather(out, t)
        return [o.tolist() for o in out]

    def halo(self, X, b: int):
        """q_y x (n + 2b) block: left halo | X | right halo (zeros at the domain ends)."""
        t, L = self.t, self.L
        qy, n = X.shape
        ext = t.zeros((qy, n + 2 * b), dtype=X.dtype, device=X.device)
        ext[:, b:b + n] = X
        if b == 0 or L.world == 1:
            return ext
        if n < b:
            raise SolverError(f"column shard of {n} columns is narrower than the halo {b}")
        ops = []
        left, right = L.rank - 1, L.rank + 1
        lrecv = t.empty((qy, b), dtype=X.dtype, device=X.device)
        rrecv = t.empty((qy, b), dtype=X.dtype, device=X.device)
        if left >= 0:
            peer = self.ranks[left]
            ops.append(self.dist.P2POp(self.dist.isend, X[:, :b].contiguous(), peer, group=self.group))
            ops.append(self.dist.P2POp(self.dist.irecv, lrecv, peer, group=self.group))
        if right < L.world:
            peer = self.ranks[right]
            ops.append(self.dist.P2POp(self.dist.isend, X[:, n - b:].contiguous(), peer, group=self.group))
            ops.append(self.dist.P2POp(self.dist.irecv, rrecv, peer, group=self.group))
        for req in self.dist.batch_isend_irecv(ops):
            req.wait()
        if left >= 0:
            ext[:, :b] = lrecv
        if right < L.world:
            ext[:, b + n:] = rrecv
        return ext

    def _all_to_all(self, send_blocks, recv_shapes, dtype, device):
        t = self.t
        send = t.cat([blk.reshape(-1) for blk in send_blocks])
        rsizes = [a * c for a, c in recv_shapes]
        recv = t.empty(sum(rsizes), dtype=dtype, device=device)
        if self.L.world == 1:
            recv.copy_(send)
        else:
            self.dist.all_to_all_single(recv, send, rsizes, [blk.numel() for blk in send_blocks],
                                        group=self.group)
        return t.split(recv, rsizes)

    def cols_to_rows(self, Xc):
        """q_y x n (column shard) -> m x q_x (row shard)."""
        L = self.L
        send = [Xc[L.row_offs[s]:L.row_offs[s] + L.row_counts[s], :] for s in range(L.world)]
        parts = self._all_to_all(send, [(L.m, L.col_counts[s]) for s in range(L.world)], Xc.dtype, Xc.device)
        return self.t.cat([p.reshape(L.m, L.col_counts[s]) for s, p in enumerate(parts)], dim=1)

    def rows_to_cols(self, Xr):
        """m x q_x (row shard) -> q_y x n (column shard)."""
        L = self.L
        send = [Xr[:, L.col_offs[s]:L.col_offs[s] + L.col_counts[s]] for s in range(L.world)]
        parts = self._all_to_all(send, [(L.row_counts[s], L.n) for s in range(L.world)], Xr.dtype, Xr.device)
        return self.t.cat([p.reshape(L.row_counts[s], L.n) for s, p in enumerate(parts)], dim=0)

    def rowsT_to_colsT(self, XrT):
        """q_x x m (transposed row shard) -> n x q_y (transposed column shard)."""
        L = self.L
        send = [XrT[L.col_offs[s]:L.col_offs[s] + L.col_counts[s], :] for s in range(L.world)]
        parts = self._all_to_all(send, [(L.n, L.row_counts[s]) for s in range(L.world)], XrT.dtype,
                                 XrT.device)
        return self.t.cat([p.reshape(L.n, L.row_counts[s]) for s, p in enumerate(parts)], dim=1)


class PeerTransposes:
    """The two transposes of the sharded preconditioner over peer memory
    (CUDA IPC mappings of the other ranks' receive buffers; NVLink stores
    between the GPUs of one node) instead of NCCL all-to-alls:

    * cols -> rows: each rank copies the row block of rank s out of its
      column shard of R straight into rank s's row buffer (P2P copies);
    * rows^T -> cols^T: fused into the GEMM that produces the data —
      X^T = P_R^-T R_rows^T is computed by ``sfb_dgemm_nt_scatter``, whose
      epilogue stores output row j (a grid column) into the column-shard
      buffer of the rank that owns column j.

    ``sync()`` after each exchange makes the peers' stores visible:
    ``"host"`` (stream synchronize + process-group barrier: the ranks only
    meet on the host, so ranks sharing one GPU never wait on each other's
    kernels) or ``"stream"`` (a one-element NCCL all-reduce on the stream,
    for one GPU per rank).  Reuse of the receive buffers across iterations is
    ordered by the scalar all-reduces of the iteration, which every rank
    joins only after its preconditioner GEMMs have read them."""

    def __init__(self, layout: Layout, backend, group=None, sync: str = "host"):
        import torch
        import torch.distributed as dist
        self.t, self.dist, self.L, self.group = torch, dist, layout, group
        self.backend = backend  # its prepared constant operands (right_T_scatter)
        if sync not in ("host", "stream"):
            raise ConfigError(f"unknown peer sync mode '{sync}'")
        self.sync_mode = sync
        L = layout
        # receive buffers: row shard of R (m x q_x) and transposed column shard (n x q_y)
        self.rows = backend.zeros(L.m, L.qx)
        self.colsT = backend.zeros(L.n, L.qy)
        self.cols = backend.zeros(L.qy, L.n)  # banded form: rows -> cols without a transpose
        mine = [self._handle(self.rows), self._handle(self.colsT), self._handle(self.cols)]
        allh = [None] * L.world
        dist.all_gather_object(allh, mine, group=group)
        self._bases = []
        self.peer_rows, self.peer_colsT, self.peer_cols = [], [], []
        for r in range(L.world):
            if r == L.rank:
                self.peer_rows.append((self.rows.data_ptr(), self.rows.stride(0)))
                self.peer_colsT.append((self.colsT.data_ptr(), self.colsT.stride(0)))
                self.peer_cols.append((self.cols.data_ptr(), self.cols.stride(0)))
                continue
            (hr, orr, ldr), (hc, oc, ldc), (hk, ok, ldk) = allh[r]
            self.peer_rows.append((self._open(hr, orr), ldr))
            self.peer_colsT.append((self._open(hc, oc), ldc))
            self.peer_cols.append((self._open(hk, ok), ldk))
        self._flag = torch.zeros(1, dtype=torch.float64, device="cuda") if sync == "stream" else None

    def _handle(self, X):
        h = (nat.C.c_ubyte * 64)()
        off = nat.C.c_ulonglong(0)
        nat.check(nat.lib().sfb_ipc_get_handle(X.data_ptr(), h, nat.C.byref(off)), "ipc handle")
        return bytes(h), int(off.value), X.stride(0)

    def _open(self, handle, offset):
        base, ptr = nat.C.c_void_p(), nat.C.c_void_p()
        nat.check(nat.lib().sfb_ipc_open((nat.C.c_ubyte * 64).from_buffer_copy(handle), offset,
                                         nat.C.byref(base), nat.C.byref(ptr)), "ipc open")
        self._bases.append(base.value)
        return ptr.value

    def close(self):
        for b in self._bases:
            nat.lib().sfb_ipc_close(b)
        self._bases = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        if self.sync_mode == "stream":  # also at world 1: one code path (a no-op NCCL kernel)
            self.dist.all_reduce(self._flag, group=self.group)
        elif self.L.world == 1:
            return
        else:
            self.t.cuda.current_stream().synchronize()
            self.dist.barrier(group=self.group)

    def cols_to_rows(self, Xc):
        """Push the row block of every rank out of this column shard (P2P copies)."""
        L = self.L
        Xc = Xc if Xc.stride(1) == 1 else Xc.contiguous()
        for s in range(L.world):
            dst, ldd = self.peer_rows[s]
            src = Xc[L.row_offs[s]:L.row_offs[s] + L.row_counts[s], :]
            nat.check(nat.lib().sfb_copy2d(dst + 8 * L.c0, ldd, src.data_ptr(), Xc.stride(0), L.row_counts[s], L.n,
                                           nat.stream()), "peer copy")
        self.sync()
        return self.rows

    def rows_to_cols(self, Xr):
        """Push every rank's column block of this row shard into its column
        buffer at this rank's row offset (P2P copies)."""
        L = self.L
        Xr = Xr if Xr.stride(1) == 1 else Xr.contiguous()
        for s in range(L.world):
            dst, ldd = self.peer_cols[s]
            src = Xr[:, L.col_offs[s]:L.col_offs[s] + L.col_counts[s]]
            nat.check(nat.lib().sfb_copy2d(dst + 8 * L.r0 * ldd, ldd, src.data_ptr(), Xr.stride(0), L.m,
                                           L.col_counts[s], nat.stream()), "peer copy")
        self.sync()
        return self.cols

    def right_T_scatter(self, RinvT, R_rows, st=None):
        """X^T = P_R^-T R_rows^T with each output row stored straight into
        its owner's transposed column shard; returns this rank's shard
        (gated on the sharded solve's status when ``st`` is given)."""
        L = self.L
        A, B = RinvT, R_rows
        if B.stride(0) % 2 or B.data_ptr() % 16:
            B = B.contiguous()
        n = L.world
        seg = (nat.C.c_int * (n + 1))(*(list(L.col_offs) + [L.qx]))
        dst = (nat.C.c_void_p * n)(*[p for p, _ in self.peer_colsT])
        ldd = (nat.C.c_int * n)(*[ld for _, ld in self.peer_colsT])
        const = getattr(self.backend, "_const", {}).get(A.data_ptr()) if st is not None else None
        if const is not None:  # the prepared P_R^-T: same product, Strassen schedule above the threshold
            nat.check(nat.lib().sfb_shard_gemm_scatter_const(st.handle.p, const.p, B.data_ptr(), B.stride(0), L.m, n,
                                                             seg, dst, ldd, L.r0, nat.stream()), "scatter gemm")
        elif st is not None:
            nat.check(nat.lib().sfb_shard_gemm_scatter(st.handle.p, A.data_ptr(), A.stride(0), B.data_ptr(),
                                                       B.stride(0), L.qx, L.m, L.qx, n, seg, dst, ldd, L.r0,
                                                       nat.stream()), "scatter gemm")
        else:
            nat.check(nat.lib().sfb_dgemm_nt_scatter(A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), L.qx,
                                                      L.m, L.qx, n, seg, dst, ldd, L.r0, nat.stream()),
                      "scatter gemm")
        self.sync()
        return self.colsT


class _DeviceSlots:
    """A device array owned by the library, seen by torch (in-place NCCL)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None}


class ShardState:
    """Device scalars of one sharded solve (sfb_shard_*): PcgState, history
    and the all-reduce slots [<W,Q>, |Q|^2, |R|^2, <Z,R>, beta]."""

    def __init__(self, max_iter: int, stop: StoppingRule):
        import torch
        L = nat.lib()
        out = nat.C.c_void_p()
        nat.check(L.sfb_shard_create(int(max_iter), stop.native_kind, float(stop.value), nat.C.byref(out)),
                  "shard state")
        self.handle = nat.Handle(out.value, L.sfb_shard_destroy)
        self.max_iter = max_iter
        self.slots = torch.as_tensor(_DeviceSlots(L.sfb_shard_slots(self.handle.p), 8), device="cuda")
        self.host_reads = 0


class CudaBackend:
    """Local compute of one rank through the C ABI (banded block operator,
    DMMA GEMMs, fused vector passes, device-resident iteration state)."""

    def __init__(self, op, precond, layout: Layout):
        import torch
        self.t = torch
        self.L = layout
        L = nat.lib()
        if not op.banded:
            raise SolverError("the sharded MO-PCG needs a banded operator")
        w, off, g, h = op.band_layout()
        self.b = (w - 1) // 2
        hl = np.ascontiguousarray(h[:, layout.c0:layout.c0 + layout.n, :])
        out = nat.C.c_void_p()
        nat.check(L.sfb_op_create_block(layout.qy, layout.n, layout.n + 2 * self.b, len(op.terms), w, off,
                                        nat.host_ptr(g), 0, nat.host_ptr(hl), nat.C.byref(out)), "block op")
        self._op = nat.Handle(out.value, L.sfb_op_destroy)
        self.banded = False
        if precond.is_identity:
            self.Linv = self.RinvT = None
        elif precond.mode == "banded":
            # SPIKE solves on the shards: the right factor along the rows of a
            # row shard (after the first transpose), the left factor along the
            # columns of a column shard (reference solvers.py:134-143)
            from .solvers import _cholesky_band
            qy, qx = layout.qy, layout.qx
            cl, cr = _cholesky_band(precond.left, qy), _cholesky_band(precond.right, qx)
            if cl is None or cr is None:
                raise SolverError("banded preconditioner mode needs symmetric positive definite "
                                  "factors with half-bandwidth <= 4")
            self.banded = True
            self.Linv = self.RinvT = None
            self._pre_rows = self._banded_pre(layout.m, qx, (0, np.ones((layout.m, 1))), cr)
            self._pre_cols = self._banded_pre(qy, layout.n, cl, (0, np.ones((layout.n, 1))))
        else:
            qy, qx = layout.qy, layout.qx
            # formed on the device and kept there (no host round trip)
            self.Linv = self.from_host(precond._inverse(precond.left, qy, left=True))
            self.RinvT = self.from_host(precond._inverse(precond.right, qx, left=False).T)
            # the two constant left operands, prepared once for the device-resident
            # iteration (Strassen leaf operands from the threshold of set_strassen_min_q
            # on; the right operands are this rank's columns / rows)
            self._const = {}
            for A, q, n_max in ((self.Linv, qy, layout.n), (self.RinvT, qx, layout.m)):
                out = nat.C.c_void_p()
                nat.check(L.sfb_const_create(A.data_ptr(), A.stride(0), q, q, max(int(n_max), 1), nat.C.byref(out)),
                          "constant operand")
                self._const[A.data_ptr()] = nat.Handle(out.value, L.sfb_const_destroy)

    # -- helpers ------------------------------------------------------------
    @staticmethod
    def _banded_pre(rows, cols, left, right):
        L = nat.lib()
        out = nat.C.c_void_p()
        nat.check(L.sfb_pre_create_banded(rows, cols, left[0], nat.host_ptr(np.ascontiguousarray(left[1])),
                                          right[0], nat.host_ptr(np.ascontiguousarray(right[1])),
                                          nat.C.byref(out)), "banded shard preconditioner")
        return nat.Handle(out.value, L.sfb_pre_destroy)

    def _pre(self, h, X, rows, cols, st=None):
        Z = self._padded(rows, cols)
        if st is not None:  # gated on the sharded solve's status
            if X.stride(0) % 2 or X.data_ptr() % 16:
                X = self.copy(X)
            nat.check(nat.lib().sfb_shard_pre_apply(st.handle.p, h.p, X.data_ptr(), X.stride(0), Z.data_ptr(),
                                                    Z.stride(0), nat.stream()), "banded shard preconditioner")
            return Z
        nat.check(nat.lib().sfb_pre_apply(h.p, X.data_ptr(), X.stride(0), Z.data_ptr(), Z.stride(0), nat.stream()),
                  "banded shard preconditioner")
        return Z

    def right_rows(self, Xr, st=None):  # Xr P_R^-1 on a row shard (m x q_x)
        return self._pre(self._pre_rows, Xr, self.L.m, self.L.qx, st)

    def left_cols(self, Xc, st=None):  # P_L^-1 Xc on a column shard (q_y x n)
        return self._pre(self._pre_cols, Xc, self.L.qy, self.L.n, st)

    def _padded(self, rows, cols):
        t = self.t
        buf = t.zeros((rows, cols + (cols % 2)), dtype=t.float64, device="cuda")
        return buf[:, :cols]

    def _padded_from(self, a):
        v = self._padded(*a.shape)
        v.copy_(self.t.from_numpy(np.ascontiguousarray(a)))
        return v

    def _gemm(self, A, Bt, M, N, K, st=None):
        C = self._padded(M, N)
        As, Bs = A, Bt
        if As.stride(0) % 2 or As.data_ptr() % 16:
            As = self._padded(*A.shape)
            As.copy_(A)
        if Bs.stride(0) % 2 or Bs.data_ptr() % 16:
            Bs = self._padded(*Bt.shape)
            Bs.copy_(Bt)
        if st is not None:  # gated on the sharded solve's status
            const = getattr(self, "_const", {}).get(As.data_ptr())
            if const is not None:  # a prepared constant operand (P_L^-1, P_R^-T)
                nat.check(nat.lib().sfb_shard_gemm_const(st.handle.p, const.p, Bs.data_ptr(), Bs.stride(0), N,
                                                         C.data_ptr(), C.stride(0), nat.stream()), "gemm")
                return C
            nat.check(nat.lib().sfb_shard_gemm(st.handle.p, As.data_ptr(), As.stride(0), Bs.data_ptr(), Bs.stride(0),
                                               M, N, K, C.data_ptr(), C.stride(0), nat.stream()), "gemm")
            return C
        nat.check(nat.lib().sfb_dgemm_nt(As.data_ptr(), As.stride(0), Bs.data_ptr(), Bs.stride(0), M, N, K,
                                         C.data_ptr(), C.stride(0), nat.stream()), "gemm")
        return C

    # -- backend interface ----------------------------------------------------
    def zeros(self, rows, cols):
        return self._padded(rows, cols)

    def from_host(self, a):
        if isinstance(a, self.t.Tensor):
            v = self._padded(*a.shape)
            v.copy_(a)
            return v
        return self._padded_from(np.asarray(a, dtype=float))

    def apply_ext(self, ext, st=None):
        L = self.L
        W = self._padded(L.qy, L.n)
        e = ext if ext.stride(1) == 1 else ext.contiguous()  # row-strided blocks are read in place
        if st is not None:  # gated on the sharded solve's status
            nat.check(nat.lib().sfb_shard_apply(st.handle.p, self._op.p, e.data_ptr(), e.stride(0), W.data_ptr(),
                                                W.stride(0), nat.stream()), "apply")
            return W
        nat.check(nat.lib().sfb_op_apply(self._op.p, e.data_ptr(), e.stride(0), W.data_ptr(), W.stride(0),
                                         nat.stream()), "apply")
        return W

    def right_T(self, R_rows, st=None):  # (P_R^-1)^T R_rows^T  : q_x x m
        return self._gemm(self.RinvT, R_rows, self.L.qx, R_rows.shape[0], self.L.qx, st)

    def left(self, XcT, st=None):  # P_L^-1 X_cols : q_y x n
        return self._gemm(self.Linv, XcT, self.L.qy, XcT.shape[0], self.L.qy, st)

    def copy(self, X):
        Y = self._padded(*X.shape)
        Y.copy_(X)
        return Y

    def update(self, U, R, Q, W, alpha):
        out = np.zeros(1)
        nat.check(nat.lib().sfb_vec_update(U.data_ptr(), R.data_ptr(), Q.data_ptr(), W.data_ptr(), U.stride(0),
                                           U.shape[0], U.shape[1], float(alpha), nat.dptr(out), nat.stream()),
                  "update")
        return float(out[0])

    def xpby(self, Q, Z, beta, first=False):
        nat.check(nat.lib().sfb_vec_xpby(Q.data_ptr(), Q.stride(0), Z.data_ptr(), Z.stride(0), Q.shape[0],
                                         Q.shape[1], float(beta), int(first), nat.stream()), "xpby")

    def dots(self, A, B, C=None, D=None):
        out = np.zeros(2)
        nat.check(nat.lib().sfb_vec_dots(A.data_ptr(), B.data_ptr(), C.data_ptr() if C is not None else None,
                                         D.data_ptr() if D is not None else None, A.stride(0), A.shape[0],
                                         A.shape[1], nat.dptr(out), nat.stream()), "dots")
        return float(out[0]), float(out[1])

    def to_host(self, X):
        return X.cpu().numpy()

    # -- device-resident iteration state (no host round trip) -----------------
    def state(self, max_iter, stop):
        return ShardState(max_iter, stop)

    def sdots(self, st, A, B, C=None, D=None, slot=0):
        nat.check(nat.lib().sfb_shard_dots(
            st.handle.p, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0),
            C.data_ptr() if C is not None else None, C.stride(0) if C is not None else 0,
            D.data_ptr() if D is not None else None, D.stride(0) if D is not None else 0,
            A.shape[0], A.shape[1], int(slot), nat.stream()), "shard dots")

    def sstart(self, st):
        nat.check(nat.lib().sfb_shard_start(st.handle.p, nat.stream()), "shard start")

    def supdate(self, st, U, R, Q, W):
        nat.check(nat.lib().sfb_shard_update(st.handle.p, U.data_ptr(), U.stride(0), R.data_ptr(), R.stride(0),
                                             Q.data_ptr(), Q.stride(0), W.data_ptr(), W.stride(0), U.shape[0],
                                             U.shape[1], nat.stream()), "shard update")

    def scontrol(self, st):
        nat.check(nat.lib().sfb_shard_control(st.handle.p, nat.stream()), "shard control")

    def sxpby(self, st, Q, Z, first=False):
        nat.check(nat.lib().sfb_shard_xpby(st.handle.p, Q.data_ptr(), Q.stride(0), Z.data_ptr(), Z.stride(0),
                                           Q.shape[0], Q.shape[1], int(first), nat.stream()), "shard xpby")

    def sresult(self, st, history=False):
        """(status, iterations, bad_iter, bad_value[, history, increments]):
        the one host synchronisation of a chunk."""
        res = nat.PcgResult()
        h = np.zeros(st.max_iter + 1) if history else None
        i = np.zeros(max(st.max_iter, 1)) if history else None
        nat.check(nat.lib().sfb_shard_result(st.handle.p, nat.C.byref(res), nat.dptr(h) if history else None,
                                             nat.dptr(i) if history else None, nat.stream()), "shard result")
        st.host_reads += 1
        out = (res.stop_reason, res.iterations, res.bad_iter, res.bad_value)
        if history:
            out += (h[:res.iterations + 1], i[:res.iterations])
        return out


_STATUS = {nat.PCG_TOLERANCE: "tolerance", nat.PCG_INCREMENT: "increment", nat.PCG_MAX_ITER: "max_iter"}


def sharded_mo_pcg(backend, comm: Comm, rhs_local, stop: StoppingRule | None = None, u0_local=None,
                   max_iter: int = 1000, identity: bool = False, keep_on_device: bool = False,
                   peer: PeerTransposes | None = None, check_every: int = 16,
                   graph: bool = False) -> SolveReport:
    """MO-PCG over column shards; same recurrences, stop logic and report as
    solvers.mo_pcg (solvers.py:365-453).  Returns this rank's columns.
    With ``peer`` the preconditioner's transposes go over peer memory
    (PeerTransposes) instead of the all-to-alls of ``comm``.

    Device-resident: alpha, beta, the history and the stop test stay in the
    backend's state, the scalar all-reduces run in place on its slots, and
    the host reads the status once every ``check_every`` iterations
    (``diagnostics["host_reads"]``); iterations issued after the stop are
    gated no-ops, so the trajectory is the per-iteration loop's.  With
    ``graph=True`` (CUDA backend with NCCL or peer-memory collectives) a
    chunk is captured once into a CUDA graph — kernels and NCCL calls — and
    replayed: capture would fail on any host synchronisation inside it."""
    stop = stop or relative_residual()
    t0 = time.perf_counter()
    L = comm.L
    b = getattr(backend, "b", 0)
    n = L.n
    st = backend.state(max_iter, stop)
    B = backend.from_host(rhs_local)
    R = backend.copy(B)
    if u0_local is not None:
        Ue = backend.zeros(L.qy, n + 2 * b)
        Ue[:, b:b + n] = backend.from_host(u0_local)
        W0 = backend.apply_ext(comm.halo_(Ue, n, b))
        U = backend.copy(Ue[:, b:b + n])
        scratch = backend.zeros(L.qy, n)
        backend.update(scratch, R, backend.zeros(L.qy, n), W0, 1.0)  # R = rhs - L(U0) (setup, not the loop)
        del Ue, W0, scratch
    else:
        U = backend.zeros(L.qy, n)
    Qe = backend.zeros(L.qy, n + 2 * b)  # the direction lives inside its halo-extended block
    Q = Qe[:, b:b + n]

    def precond(Rk, st=None):  # st: gate the heavy kernels on the solve's status
        if identity:
            return backend.copy(Rk)
        if getattr(backend, "banded", False):  # SPIKE form: right solves on rows, left solves on columns
            ex = peer if peer is not None else comm
            return backend.left_cols(ex.rows_to_cols(backend.right_rows(ex.cols_to_rows(Rk), st=st)), st=st)
        if peer is not None:  # transposes over peer memory, the second fused into the GEMM
            return backend.left(peer.right_T_scatter(backend.RinvT, peer.cols_to_rows(Rk), st=st), st=st)
        XrT = backend.right_T(comm.cols_to_rows(Rk), st=st)
        return backend.left(comm.rowsT_to_colsT(XrT), st=st)

    # setup (solvers.py:389-420): |R_0|, Z_0, <Z_0, R_0>, Q_0 = Z_0
    Z = precond(R)
    backend.sdots(st, R, R, Z, R, slot=2)
    comm.allreduce_(st.slots[2:4])
    backend.sstart(st)
    backend.sxpby(st, Q, Z, first=True)
    def chunk(size):
        for _ in range(size):
            W = backend.apply_ext(comm.halo_(Qe, n, b), st=st)
            backend.sdots(st, W, Q, Q, Q, slot=0)  # <W,Q>, |Q|^2
            comm.allreduce_(st.slots[0:2])
            backend.supdate(st, U, R, Q, W)  # alpha; U, R; |R|^2 -> slot 2
            Z = precond(R, st)  # computed before the stop test: result-identical
            backend.sdots(st, Z, R, slot=3)
            comm.allreduce_(st.slots[2:4])
            backend.scontrol(st)  # history, increment, stop test, beta
            backend.sxpby(st, Q, Z)

    # chunks of 1, 2, 4, ... check_every iterations: short solves (an IMEX
    # step's few iterations) read the status early; iterations issued past the
    # stop skip their GEMMs / SPIKE / band passes (gated) and cost only their
    # communication
    full = max(1, check_every)
    size = 1
    status = backend.sresult(st)[0]
    replay = None
    while status == nat.PCG_RUNNING:
        if replay is not None:
            replay.replay()
        else:
            chunk(size)  # eager (the first full-size chunk also does every kernel's first-launch setup)
            if graph and size == full:
                import torch
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    chunk(full)  # captured, not executed
                replay = g
            size = min(2 * size, full)
        status = backend.sresult(st)[0]
    status, iters, bad_iter, bad_value, hist, incs = backend.sresult(st, history=True)
    if status == nat.PCG_INDEFINITE:
        raise OperatorError("operator is not positive definite along a search direction "
                            f"(<L(Q), Q> = {bad_value:.3e} at iteration {bad_iter})")
    if status == nat.PCG_NONFINITE:
        raise SolverError(f"mo_pcg residual became non-finite at iteration {bad_iter}")
    return SolveReport(solution=U if keep_on_device else backend.to_host(U), method="mo-pcg-sharded",
                       iterations=iters, residual_history=np.asarray(hist), stop_reason=_STATUS[status],
                       wall_time=time.perf_counter() - t0,
                       diagnostics={"dense_grid_matrices": 5, "increments": np.asarray(incs),
                                    "stopping_rule": stop.describe(), "world": L.world,
                                    "columns": (L.c0, L.c0 + L.n), "host_reads": st.host_reads,
                                    "check_every": check_every, "graph": replay is not None})


# =========================================================================
# Column-sharded IMEX heat (cfg4 across GPUs, SURVEY §8 e)
# =========================================================================
#
# imex_euler_heat (reference timestepping.py:126-159) with U column-sharded.
# Per step: the b_rhs-column halo of U; the block rhs map W = expand(U) +
# tau g(t_k) F (the fused heat loader of the banded map kernel on the
# halo-extended block, with this rank's static slice of F); the blow-up
# checks reduced over the ranks; the sharded MO-PCG warm-started from U; the
# increment norm reduced over the ranks.  Block coordinates: input column k'
# of the map is full-grid column c0 + cs - b + k' (cs = 1 for Dirichlet),
# i.e. interior column c0 - b + k', so the halo-extended block of U is read
# with no column shift and zero halos at the domain ends.


class CudaShardedHeatStepper:
    """Local compute of the column-sharded heat step through the C ABI."""

    def __init__(self, x, y, d_u, tau, lumped, inner, source, layout: Layout):
        from .fem1d import BCKind
        from .operators import parabolic_operator
        from .timestepping import SeparableSource, _parabolic_precond
        if not isinstance(source, SeparableSource):
            raise ConfigError("the column-sharded heat driver evaluates the source on the device: "
                              "pass a SeparableSource")
        if inner.method != "mo-pcg" or inner.precond == "two_term":
            raise ConfigError("the column-sharded heat driver runs MO-PCG with the reference preconditioner")
        import torch
        self.t, self.L = torch, layout
        op, rhs_of = parabolic_operator(x, y, d_u, tau, lumped=lumped)
        pre = _parabolic_precond(x, y, d_u, tau, lumped, inner, op)
        self.backend = CudaBackend(op, pre, layout)
        self.g = source.time_factor
        F = np.asarray(source.F, dtype=float)
        if F.shape != rhs_of.in_shape:
            raise ConfigError(f"separable source must cover the full node grid {rhs_of.in_shape}")
        self.rs = 1 if y.basis.bc is BCKind.DIRICHLET else 0
        cs = 1 if x.basis.bc is BCKind.DIRICHLET else 0
        w, goff, g, hoff, h = rhs_of.layout()
        self.b = max(0, cs - hoff, hoff - cs + w - 1)
        n, c0, b = layout.n, layout.c0, self.b
        ncols = n + 2 * b
        Fb = np.zeros((F.shape[0], ncols))  # full-grid columns c0 + cs - b ... (zero outside the grid)
        lo = c0 + cs - b
        a0, a1 = max(lo, 0), min(lo + ncols, F.shape[1])
        Fb[:, a0 - lo:a1 - lo] = F[:, a0:a1]
        self.F = self.backend.from_host(Fb)
        hl = np.ascontiguousarray(h[c0:c0 + n])
        out = nat.C.c_void_p()
        nat.check(nat.lib().sfb_map_create(layout.qy, n, F.shape[0], ncols, w, goff,
                                           nat.host_ptr(np.ascontiguousarray(g)), w, hoff - cs + b,
                                           nat.host_ptr(hl), nat.C.byref(out)), "block rhs map")
        self._map = nat.Handle(out.value, nat.lib().sfb_map_destroy)

    def to_local(self, a):
        L = self.L
        if nat.is_device(a):
            return self.backend.from_host(a[:, L.c0:L.c0 + L.n])
        return self.backend.from_host(np.asarray(a, dtype=float)[:, L.c0:L.c0 + L.n])

    def rhs(self, Ue, c):
        """local rhs of W = expand(U) + c F and local [max|W|, #non-finite(W)]."""
        out = self.backend.zeros(self.L.qy, self.L.n)
        chk = np.zeros(2)
        nat.check(nat.lib().sfb_map_apply_heat(self._map.p, Ue.data_ptr(), Ue.stride(0), self.rs, 0, float(c),
                                               self.F.data_ptr(), self.F.stride(0), out.data_ptr(), out.stride(0),
                                               nat.dptr(chk), nat.stream()), "heat rhs")
        return out, chk

    def norms(self, A, B):
        """local {sum (A-B)^2, max|A|, #non-finite(A), sum A^2}."""
        out = np.zeros(4)
        nat.check(nat.lib().sfb_diff_norm(A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), A.shape[0],
                                          A.shape[1], nat.dptr(out), nat.stream()), "norm")
        return [out[0] ** 2, out[1], out[2], out[3] ** 2]

    def host(self, X):
        return nat.to_host(X)


def sharded_imex_heat(domain, x, y, d_u: float, source, u0, grid, inner=None, lumped: bool = False,
                      comm: Comm | None = None, stepper=None, peer_sync: str | None = None,
                      graph: bool = False):
    """imex_euler_heat (timestepping.py:126-159) with U column-sharded over
    the ranks of ``comm`` (SURVEY §8 e; cfg4 at 1/2/4/8 GPUs).  ``u0`` is the
    full initial state (each rank keeps its columns); ``source`` a
    SeparableSource.  Returns this rank's columns in ``final``; increments
    and iteration counts are global and equal on all ranks.  ``peer_sync``
    ("stream" for one GPU per rank) routes the preconditioner's transposes
    over peer memory."""
    from .timestepping import BLOWUP_LIMIT, BlowUpError, InnerSolver, Trajectory, _step_setup
    inner = inner or InnerSolver()
    _step_setup(inner)
    tau = grid.tau
    if comm is None:
        import torch.distributed as dist
        comm = Comm(Layout(y.q, x.q, dist.get_world_size(), dist.get_rank()), "cuda")
    L = comm.L
    st = stepper or CudaShardedHeatStepper(x, y, d_u, tau, lumped, inner, source, L)
    be = st.backend
    peer = PeerTransposes(L, be, sync=peer_sync) if peer_sync else None
    stop = inner.stopping(tau)
    U = st.to_local(u0)
    Ue = be.zeros(L.qy, L.n + 2 * st.b)
    n = grid.n_steps
    incs = np.empty(n)
    iters = np.empty(n, dtype=int)
    try:
        for k in range(n):
            Ue[:, st.b:st.b + L.n] = U
            rhs, chk = st.rhs(comm.halo_(Ue, L.n, st.b), tau * float(st.g(k * tau)))
            mx, = _allreduce_max(comm, [chk[0]])
            cnt, = comm.allreduce([chk[1]])
            if cnt > 0 or mx > BLOWUP_LIMIT:
                raise BlowUpError(k, "u", st.host(U))
            rep = sharded_mo_pcg(be, comm, rhs, stop=stop, u0_local=U, max_iter=inner.max_iter,
                                 keep_on_device=True, peer=peer, graph=graph)
            if rep.stop_reason == "max_iter" and stop.kind != "budget":
                raise SolverError(f"inner PCG did not converge in {inner.max_iter} iterations")
            loc = st.norms(rep.solution, U)
            dd, bad = comm.allreduce([loc[0], loc[2]])
            mx, = _allreduce_max(comm, [loc[1]])
            if bad > 0 or mx > BLOWUP_LIMIT:
                raise BlowUpError(k, "u", st.host(U))
            incs[k] = math.sqrt(dd)
            iters[k] = rep.iterations
            U = rep.solution
    finally:
        if peer is not None:
            peer.close()
    return Trajectory(final=(st.host(U),), increments=incs, iterations=iters, times=(1 + np.arange(n)) * tau,
                      diagnostics={"world": L.world, "columns": (L.c0, L.c0 + L.n)})


# =========================================================================
# Species-parallel IMEX for the two-species reaction-diffusion system
# =========================================================================
#
# Within one IMEX step the two species' implicit solves are independent: both
# right-hand sides are built from the state at the start of the step
# (timestepping.py:200-211), so species u and species v can be solved on
# different GPUs at the same time.  Rank r owns species r.  Per step:
#
#   1. rhs_r = weak rhs of S_r + tau rho kin_r(U, V)     (local, both states held)
#   2. S_r' = MO-PCG solve, warm started from S_r        (local)
#   3. one all-gather of 6 status doubles per rank: the blow-up / convergence
#      flags are then resolved in the reference's order (u rhs, u solve,
#      v rhs, v solve; timestepping.py:202-209) on every rank, so all ranks
#      raise the same exception at the same step;
#   4. one all-gather of the new states (q^2 doubles per rank) so every rank
#      holds (U', V') for the next step's kinetics.
#
# The result is bit-identical to the single-GPU driver (same kernels on the
# same inputs in the same order; only the placement differs).


class SpeciesComm:
    """Collectives of the species-parallel step over torch.distributed
    (NCCL with CUDA tensors, or gloo with CPU tensors)."""

    def __init__(self, device, group=None):
        import torch
        import torch.distributed as dist
        self.t, self.dist = torch, dist
        self.device = device
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def gather_status(self, vals):
        t = self.t.tensor(vals, dtype=self.t.float64, device=self.device)
        out = [self.t.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [o.tolist() for o in out]

    def exchange(self, own):
        """all-gather of one state per rank -> the list of states by rank."""
        own = own.contiguous()
        out = [self.t.empty_like(own) for _ in range(self.world)]
        self.dist.all_gather(out, own, group=self.group)
        out[self.rank] = own
        return out


class CudaSpeciesStepper:
    """One species' IMEX step on this rank's GPU through the C ABI: the fused
    rhs+kinetics banded map, the device MO-PCG, the device norms — the same
    calls the single-GPU driver (timestepping.imex_euler_rds) makes."""

    def __init__(self, x, y, d, tau, rho, kinetics, inner, lumped, species):
        from .models import DIBKinetics
        from .timestepping import _step_system
        self.species = species
        self.tau, self.rho = tau, rho
        self.inner = inner
        # the single-GPU driver's bounded step cache: repeated calls (one IMEX
        # step per call) reuse the operator, its preconditioner's dense
        # inverses and the solver workspaces
        self.op, self.rhs_of, self.pre = _step_system(x, y, d, tau, lumped, inner)
        self.stop = inner.stopping(tau)
        self.kinetics = kinetics
        self.device_kin = isinstance(kinetics, DIBKinetics)
        self.kp = kinetics.params.device_params() if self.device_kin else None

    def to_local(self, a):
        return nat.to_device(a).clone()

    def rhs(self, U, V):
        if self.device_kin:
            return self.rhs_of.dib(U, V, self.species, self.tau * self.rho, self.kp)
        Uh, Vh = nat.to_host(U), nat.to_host(V)
        rate = np.asarray(self.kinetics[self.species](Uh, Vh))
        W = (Uh if self.species == 0 else Vh) + self.tau * self.rho * rate
        fin = np.isfinite(W)
        chk = (float(np.max(np.abs(W[fin]))) if fin.any() else 0.0, float((~fin).sum()))
        return self.rhs_of(nat.to_device(W)), chk

    def solve(self, rhs, warm):
        """-> (new state, iterations, converged)."""
        from .solvers import mo_pcg
        from .timestepping import _direct
        if self.inner.method == "direct":
            sol, it = _direct(self.op, rhs, warm)
            return sol, it, True
        rep = mo_pcg(self.op, rhs, precond=self.pre, stop=self.stop, u0=warm, max_iter=self.inner.max_iter)
        return rep.solution, rep.iterations, rep.stop_reason != "max_iter" or self.stop.kind == "budget"

    def norms(self, A, B):
        from .timestepping import _norms
        return [float(v) for v in _norms(A, B)]

    def host(self, X):
        return nat.to_host(X)


def species_parallel_imex_rds(domain, x, y, d_u: float, d_v: float, kinetics, rho: float, state0, grid,
                              inner=None, lumped: bool = False, snapshot_every: int = 0,
                              steady_eps: float = 1e-8, comm: SpeciesComm | None = None,
                              stepper_factory=None):
    """imex_euler_rds (timestepping.py:162-220) with species r solved on rank r
    of a 2-rank group.  Every rank returns the same Trajectory.

    ``stepper_factory(x, y, d, tau, rho, kinetics, inner, lumped, species)``
    builds the local compute (default: ``CudaSpeciesStepper``)."""
    from .timestepping import BLOWUP_LIMIT, BlowUpError, InnerSolver, Trajectory, _step_setup
    if d_u <= 0 or d_v <= 0 or rho <= 0:
        raise ConfigError("d_u, d_v and rho must be positive")
    from .fem1d import BCKind
    if x.basis.bc is not BCKind.NEUMANN:
        raise ConfigError("the reaction-diffusion stepper expects zero-flux BCs")
    inner = inner or InnerSolver()
    _step_setup(inner)
    if comm is None:
        import torch
        comm = SpeciesComm("cuda" if torch.cuda.is_available() else "cpu")
    if comm.world != 2:
        raise ConfigError(f"species-parallel stepping needs a group of 2 ranks (one per species), got {comm.world}")
    s = comm.rank
    factory = stepper_factory or CudaSpeciesStepper
    tau = grid.tau
    st = factory(x, y, (d_u, d_v)[s], tau, rho, kinetics, inner, lumped, s)
    S = [st.to_local(state0[0]), st.to_local(state0[1])]
    n = grid.n_steps
    incs = np.empty((n, 2))
    iters = np.empty((n, 2), dtype=int)
    snaps = []
    steady = None
    names = ("u", "v")
    for k in range(n):
        rhs, chk = st.rhs(S[0], S[1])
        rhs_bad = float(chk[1] > 0 or chk[0] > BLOWUP_LIMIT)
        conv, sol_bad, it, nrm = 1.0, 0.0, 0, [0.0, 0.0, 0.0, 0.0]
        new = None
        if not rhs_bad:
            new, it, ok = st.solve(rhs, S[s])
            conv = float(ok)
            if ok:
                nrm = st.norms(new, S[s])
                sol_bad = float(nrm[2] > 0 or nrm[1] > BLOWUP_LIMIT)
        stat = comm.gather_status([rhs_bad, conv, sol_bad, float(it), nrm[0], nrm[3]])
        for r in range(2):  # the reference's order of checks
            if stat[r][0]:
                raise BlowUpError(k, names[r], (st.host(S[0]), st.host(S[1])))
            if not stat[r][1]:
                raise SolverError(f"inner PCG did not converge in {inner.max_iter} iterations")
            if stat[r][2]:
                raise BlowUpError(k, names[r], (st.host(S[0]), st.host(S[1])))
        incs[k] = (stat[0][4], stat[1][4])
        iters[k] = (int(stat[0][3]), int(stat[1][3]))
        S = comm.exchange(new)
        if steady is None and np.all(incs[k] <= steady_eps * max(stat[0][5], 1e-300)):
            steady = k
        if snapshot_every and ((k + 1) % snapshot_every == 0 or k == n - 1):
            snaps.append((k + 1, st.host(S[0]), st.host(S[1])))
    return Trajectory(final=(st.host(S[0]), st.host(S[1])), increments=incs, iterations=iters,
                      times=(1 + np.arange(n)) * tau, steady_step=steady, snapshots=snaps,
                      diagnostics={"species_rank": s, "world": comm.world})


# =========================================================================
# Column-sharded IMEX for the two-species reaction-diffusion system (cfg5)
# =========================================================================
#
# Both species' states are column-sharded like the MO-PCG iterates.  Per step
# (timestepping.py:200-218):
#
#   1. b_rhs-column halos of U and V (zero for the lumped P1 rhs, whose right
#      factor M0 is diagonal);
#   2. per species: rhs = G_full (S + tau rho kin(U, V)) H_full^T on the local
#      block (the fused DIB map kernel reading the halo-extended block), the
#      blow-up check reduced over ranks (max, count), then the column-sharded
#      MO-PCG warm started from the local state, then the increment / blow-up
#      norms reduced over ranks;
#   3. steady-state test and snapshots on the reduced norms.
#
# Every rank takes the same decisions from the same reduced scalars, so all
# ranks raise the same exception at the same step.


def _allreduce_max(comm, vals):
    """max over ranks through the sum-allreduce of Comm: gather by slot."""
    L = comm.L
    slots = [0.0] * (len(vals) * L.world)
    slots[L.rank * len(vals):(L.rank + 1) * len(vals)] = list(vals)
    tot = comm.allreduce(slots)
    return [max(tot[r * len(vals) + i] for r in range(L.world)) for i in range(len(vals))]


class CudaShardedDibStepper:
    """Local compute of the column-sharded DIB step: per-species CudaBackend
    (block operator, inverse-form DMMA preconditioner, vector passes) and the
    block DIB rhs map, all through the C ABI."""

    def __init__(self, x, y, d_u, d_v, tau, rho, kinetics, inner, lumped, layout: Layout, species=(0, 1)):
        from .models import DIBKinetics
        from .operators import parabolic_operator
        from .timestepping import _parabolic_precond
        if not isinstance(kinetics, DIBKinetics):
            raise ConfigError("the column-sharded DIB driver evaluates the kinetics on the device: "
                              "pass a DIBKinetics pair")
        if inner.method != "mo-pcg" or inner.precond == "two_term":
            raise ConfigError("the column-sharded DIB driver runs MO-PCG with the reference preconditioner")
        self.L = layout
        self.tau_rho = tau * rho
        self.kp = np.ascontiguousarray(kinetics.params.device_params(), dtype=float)
        self.backends = [None, None]
        for sp, d in enumerate((d_u, d_v)):
            op, rhs_of = parabolic_operator(x, y, d, tau, lumped=lumped)
            if sp in species:
                pre = _parabolic_precond(x, y, d, tau, lumped, inner, op)
                self.backends[sp] = CudaBackend(op, pre, layout)
        w, goff, g, hoff, h = rhs_of.layout()
        self.b = max(0, -hoff, hoff + w - 1)
        n = layout.n
        hl = np.ascontiguousarray(h[layout.c0:layout.c0 + n])
        out = nat.C.c_void_p()
        nat.check(nat.lib().sfb_map_create(layout.qy, n, layout.qy, n + 2 * self.b, w, goff,
                                           nat.host_ptr(np.ascontiguousarray(g)), w, hoff + self.b,
                                           nat.host_ptr(hl), nat.C.byref(out)), "block rhs map")
        self._map = nat.Handle(out.value, nat.lib().sfb_map_destroy)

    def _be(self):
        return self.backends[0] if self.backends[0] is not None else self.backends[1]

    def to_local(self, a):
        L = self.L
        if nat.is_device(a):
            return self._be().from_host(a[:, L.c0:L.c0 + L.n])
        return self._be().from_host(np.asarray(a, dtype=float)[:, L.c0:L.c0 + L.n])

    def rhs(self, species, extU, extV):
        be = self._be()
        U, V = extU.contiguous(), extV.contiguous()
        out = be.zeros(self.L.qy, self.L.n)
        chk = np.zeros(2)
        nat.check(nat.lib().sfb_map_apply_dib(self._map.p, U.data_ptr(), V.data_ptr(), U.stride(0), int(species),
                                              self.tau_rho, nat.dptr(self.kp), out.data_ptr(), out.stride(0),
                                              nat.dptr(chk), nat.stream()), "dib rhs")
        return out, chk

    def norms(self, A, B):
        """local {sum (A-B)^2, max|A|, #non-finite(A), sum A^2}."""
        out = np.zeros(4)
        nat.check(nat.lib().sfb_diff_norm(A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), A.shape[0],
                                          A.shape[1], nat.dptr(out), nat.stream()), "norm")
        return [out[0] ** 2, out[1], out[2], out[3] ** 2]

    def host(self, X):
        return nat.to_host(X)


_STEPPERS: dict = {}  # per-rank setup of the sharded DIB drivers, reused across calls


def _cached_dib_stepper(x, y, d_u, d_v, tau, rho, kinetics, inner, lumped, layout: Layout, species=(0, 1)):
    """CudaShardedDibStepper of this rank, built once per (grids, coefficients,
    inner solver, layout, species): its block operators, dense preconditioner
    inverses and block rhs map are reused by later calls (one IMEX step per
    call in the benchmark).  Keyed weakly on the direction sets; at most four
    entries are kept."""
    import weakref
    kp = tuple(np.asarray(kinetics.params.device_params(), dtype=float).tolist()) \
        if hasattr(kinetics, "params") else id(kinetics)
    key = (id(x), id(y), float(d_u), float(d_v), float(tau), float(rho), kp, bool(lumped), inner.method,
           inner.precond, inner.precond_mode, layout.qy, layout.qx, layout.world, layout.rank, tuple(species))
    e = _STEPPERS.get(key)
    if e is not None and e[0]() is x and e[1]() is y:
        return e[2]
    st = CudaShardedDibStepper(x, y, d_u, d_v, tau, rho, kinetics, inner, lumped, layout, species=species)
    while len(_STEPPERS) >= 4:
        _STEPPERS.pop(next(iter(_STEPPERS)))
    _STEPPERS[key] = (weakref.ref(x), weakref.ref(y), st)
    return st


def sharded_imex_rds(domain, x, y, d_u: float, d_v: float, kinetics, rho: float, state0, grid, inner=None,
                     lumped: bool = False, snapshot_every: int = 0, steady_eps: float = 1e-8,
                     comm: Comm | None = None, stepper=None):
    """imex_euler_rds (timestepping.py:162-220) with both species' states
    column-sharded over the ranks of ``comm`` (SURVEY §8 e).  ``state0`` is
    the full pair (each rank keeps its columns).  Returns this rank's columns
    in ``final`` / ``snapshots`` / ``BlowUpError.state``; increments,
    iteration counts and the steady step are global and equal on all ranks."""
    from .fem1d import BCKind
    from .timestepping import BLOWUP_LIMIT, BlowUpError, InnerSolver, Trajectory, _step_setup
    if d_u <= 0 or d_v <= 0 or rho <= 0:
        raise ConfigError("d_u, d_v and rho must be positive")
    if x.basis.bc is not BCKind.NEUMANN:
        raise ConfigError("the reaction-diffusion stepper expects zero-flux BCs")
    inner = inner or InnerSolver()
    _step_setup(inner)
    tau = grid.tau
    if comm is None:
        import torch.distributed as dist
        comm = Comm(Layout(y.q, x.q, dist.get_world_size(), dist.get_rank()), "cuda")
    L = comm.L
    st = stepper or _cached_dib_stepper(x, y, d_u, d_v, tau, rho, kinetics, inner, lumped, L)
    stop = inner.stopping(tau)
    S = [st.to_local(state0[0]), st.to_local(state0[1])]
    n = grid.n_steps
    incs = np.empty((n, 2))
    iters = np.empty((n, 2), dtype=int)
    snaps = []
    steady = None
    names = ("u", "v")
    for k in range(n):
        ext = (comm.halo(S[0], st.b), comm.halo(S[1], st.b))
        last = lambda: (st.host(S[0]), st.host(S[1]))  # noqa: E731
        new, sq = [None, None], [None, None]
        for sp in (0, 1):
            rhs, chk = st.rhs(sp, *ext)
            mx, = _allreduce_max(comm, [chk[0]])
            cnt, = comm.allreduce([chk[1]])
            if cnt > 0 or mx > BLOWUP_LIMIT:
                raise BlowUpError(k, names[sp], last())
            rep = sharded_mo_pcg(st.backends[sp], comm, rhs, stop=stop, u0_local=S[sp], max_iter=inner.max_iter,
                                 keep_on_device=True)
            if rep.stop_reason == "max_iter" and stop.kind != "budget":
                raise SolverError(f"inner PCG did not converge in {inner.max_iter} iterations")
            loc = st.norms(rep.solution, S[sp])
            dd, bad, nn = comm.allreduce([loc[0], loc[2], loc[3]])
            mx, = _allreduce_max(comm, [loc[1]])
            if bad > 0 or mx > BLOWUP_LIMIT:
                raise BlowUpError(k, names[sp], last())
            new[sp], sq[sp] = rep.solution, nn
            incs[k, sp] = math.sqrt(dd)
            iters[k, sp] = rep.iterations
        S = new
        if steady is None and np.all(incs[k] <= steady_eps * max(math.sqrt(sq[0]), 1e-300)):
            steady = k
        if snapshot_every and ((k + 1) % snapshot_every == 0 or k == n - 1):
            snaps.append((k + 1, st.host(S[0]), st.host(S[1])))
    return Trajectory(final=(st.host(S[0]), st.host(S[1])), increments=incs, iterations=iters,
                      times=(1 + np.arange(n)) * tau, steady_step=steady, snapshots=snaps,
                      diagnostics={"world": L.world, "columns": (L.c0, L.c0 + L.n)})


# =========================================================================
# Species groups x column shards (cfg5 at 4 / 8 GPUs, SURVEY §8 e)
# =========================================================================
#
# World 2G: ranks [0, G) solve species u, ranks [G, 2G) species v, each group
# column-sharded over its G ranks with identical layouts, so rank r's
# partner r +- G owns the same columns of the other species.  Per step:
#
#   1. halo of the own species inside the group; the halo-extended block is
#      swapped with the partner (one send/recv of q x (n + 2b) doubles): the
#      pointwise DIB kinetics of the rhs need both species at the same nodes;
#   2. the rhs blow-up checks of both species, all-gathered over the world
#      (one tiny collective), resolved in the reference's order;
#   3. the own species' column-sharded MO-PCG inside the group;
#   4. the solve outcomes and increment norms, all-gathered over the world,
#      resolved in the reference's order (u rhs, u solve, v rhs, v solve).


def _group_status(vals_by_rank, G, g):
    """Rows of group g from an all-gathered status table."""
    return vals_by_rank[g * G:(g + 1) * G]


_GROUPS: dict = {}


def _species_groups(world: int, G: int):
    """The two species groups [0, G) and [G, 2G) of the default process group,
    created once per default group (communicator set-up is expensive and
    must not sit in every call; every rank calls new_group in the same order)."""
    import torch.distributed as dist
    key = (id(dist.distributed_c10d._get_default_group()), world, G)
    g = _GROUPS.get(key)
    if g is None:
        _GROUPS.clear()  # groups of a destroyed default group are dead
        g = _GROUPS[key] = [dist.new_group(list(range(k * G, (k + 1) * G))) for k in (0, 1)]
    return g


def grouped_imex_rds(domain, x, y, d_u: float, d_v: float, kinetics, rho: float, state0, grid, inner=None,
                     lumped: bool = False, snapshot_every: int = 0, steady_eps: float = 1e-8, device=None,
                     stepper_factory=None, comm_factory=None):
    """imex_euler_rds (timestepping.py:162-220) with species g on the rank
    group g (2 groups of G = world / 2 ranks), each column-sharded.  Returns
    this rank's columns of both species (``final``, ``snapshots``,
    ``BlowUpError.state``); increments, iteration counts and the steady step
    are global and equal on all ranks.

    ``stepper_factory(layout, species)`` / ``comm_factory(layout, group,
    ranks)`` replace the CUDA stepper / torch.distributed collectives (tests)."""
    import torch
    import torch.distributed as dist

    from .fem1d import BCKind
    from .timestepping import BLOWUP_LIMIT, BlowUpError, InnerSolver, Trajectory, _step_setup
    if d_u <= 0 or d_v <= 0 or rho <= 0:
        raise ConfigError("d_u, d_v and rho must be positive")
    if x.basis.bc is not BCKind.NEUMANN:
        raise ConfigError("the reaction-diffusion stepper expects zero-flux BCs")
    inner = inner or InnerSolver()
    _step_setup(inner)
    world, rank = dist.get_world_size(), dist.get_rank()
    if world % 2:
        raise ConfigError(f"species groups need an even number of ranks, got {world}")
    G = world // 2
    g, r = divmod(rank, G)
    partner = (1 - g) * G + r
    groups = _species_groups(world, G)
    L = Layout(y.q, x.q, G, r)
    device = device or ("cuda" if torch.cuda.is_available() else "cpu")
    ranks = list(range(g * G, (g + 1) * G))
    comm = comm_factory(L, groups[g], ranks) if comm_factory else Comm(L, device, group=groups[g], ranks=ranks)
    tau = grid.tau
    st = stepper_factory(L, g) if stepper_factory else \
        _cached_dib_stepper(x, y, d_u, d_v, tau, rho, kinetics, inner, lumped, L, species=(g,))
    stop = inner.stopping(tau)
    own = st.to_local(state0[g])
    other = st.to_local(state0[1 - g])  # refreshed by the swap every step
    n = grid.n_steps
    incs = np.empty((n, 2))
    iters = np.empty((n, 2), dtype=int)
    snaps = []
    steady = None
    names = ("u", "v")

    gather = comm.gather_world

    def swap(ext):
        return comm.sendrecv(ext, partner)

    def centre(ext):
        return ext[:, st.b:st.b + L.n]

    def pair():
        return (st.host(own), st.host(other)) if g == 0 else (st.host(other), st.host(own))

    for k in range(n):
        ext_own = comm.halo(own, st.b)
        ext_other = swap(ext_own)
        other = centre(ext_other).contiguous()
        ext = (ext_own, ext_other) if g == 0 else (ext_other, ext_own)
        rhs, chk = st.rhs(g, *ext)
        tab = gather([chk[0], chk[1]])
        rhs_bad = []
        for sp in (0, 1):
            rows = _group_status(tab, G, sp)
            rhs_bad.append(max(v[0] for v in rows) > BLOWUP_LIMIT or sum(v[1] for v in rows) > 0)
        # the reference checks u's rhs before anything else, v's rhs only after u's solve
        if rhs_bad[0]:
            raise BlowUpError(k, "u", pair())
        ok, its, loc, new = 1.0, 0, [0.0, 0.0, 0.0, 0.0], None
        if not rhs_bad[g]:
            rep = sharded_mo_pcg(st.backends[g], comm, rhs, stop=stop, u0_local=own, max_iter=inner.max_iter,
                                 keep_on_device=True)
            ok, its, new = float(rep.stop_reason != "max_iter" or stop.kind == "budget"), rep.iterations, rep.solution
            if ok:
                loc = st.norms(new, own)
        tab = gather([ok, float(its), loc[0], loc[1], loc[2], loc[3]])
        res = []
        for sp in (0, 1):
            rows = _group_status(tab, G, sp)
            res.append({"ok": all(v[0] for v in rows), "its": int(rows[0][1]),
                        "bad": sum(v[4] for v in rows) > 0 or max(v[3] for v in rows) > BLOWUP_LIMIT,
                        "inc": math.sqrt(sum(v[2] for v in rows)), "nrm": math.sqrt(sum(v[5] for v in rows))})
        for sp in (0, 1):  # u solve, v rhs, v solve
            if sp == 1 and rhs_bad[1]:
                raise BlowUpError(k, "v", pair())
            if not res[sp]["ok"]:
                raise SolverError(f"inner PCG did not converge in {inner.max_iter} iterations")
            if res[sp]["bad"]:
                raise BlowUpError(k, names[sp], pair())
        incs[k] = (res[0]["inc"], res[1]["inc"])
        iters[k] = (res[0]["its"], res[1]["its"])
        own = new
        if steady is None and np.all(incs[k] <= steady_eps * max(res[0]["nrm"], 1e-300)):
            steady = k
        last = k == n - 1
        if (snapshot_every and ((k + 1) % snapshot_every == 0 or last)) or last:
            other = centre(swap(comm.halo(own, st.b))).contiguous()
            if snapshot_every and ((k + 1) % snapshot_every == 0 or last):
                snaps.append((k + 1, *pair()))
    fin = pair()
    return Trajectory(final=fin, increments=incs, iterations=iters, times=(1 + np.arange(n)) * tau,
                      steady_step=steady, snapshots=snaps,
                      diagnostics={"world": world, "species_group": g, "columns": (L.c0, L.c0 + L.n)})
