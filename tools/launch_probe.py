"""Back-to-back launch timing of single kernels (stream launches, no graph).

    python tools/launch_probe.py [N]

Compares per-launch time of the banded operator, the vector update and the
banded preconditioner with their ncu durations to expose launch gaps.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2109_01173_b200 as pb  # noqa: E402
from paper_2109_01173_b200 import _native as nat  # noqa: E402
from paper_2109_01173_b200 import workloads as wl  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
w = wl.cfg3(N=N)
qy, qx = w.op.shape
L = nat.lib()
s = torch.cuda.current_stream().cuda_stream
U = torch.randn(qy, qx, dtype=torch.float64, device="cuda")
W = torch.empty_like(U)
h = w.op.native()


def timeit(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


print(f"N={N} op.apply (band kernel)      {timeit(lambda: L.sfb_op_apply(h, U.data_ptr(), qx, W.data_ptr(), qx, s)):8.1f} us")
pre = pb.make_preconditioner("elliptic_xnormal", w.x, w.y, mode="banded")
ph = pre.native(w.op.shape)
print(f"N={N} precond banded (sfb_pre_apply) {timeit(lambda: L.sfb_pre_apply(ph, U.data_ptr(), qx, W.data_ptr(), qx, s)):8.1f} us")
out = np.zeros(1)
Q = torch.randn_like(U)
R = torch.randn_like(U)


def upd():
    L.sfb_vec_update(U.data_ptr(), R.data_ptr(), Q.data_ptr(), W.data_ptr(), qx, qy, qx, 1e-9, nat.dptr(out), s)


print(f"N={N} vec update (host-synchronous)  {timeit(upd):8.1f} us")
