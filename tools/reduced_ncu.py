"""A few reduced solves (cfg1 or cfg2) for an ncu launch list, plus host-side
timings of the layers of one solve.

    python tools/reduced_ncu.py [cfg1|cfg2] [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2109_01173_b200 as pb  # noqa: E402
from paper_2109_01173_b200 import _native as nat  # noqa: E402
from paper_2109_01173_b200 import workloads as wl  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = wl.CONFIGS[name]()
cache = pb.build_spectral_cache(w.op)
cache.native()
B = torch.from_numpy(w.rhs).cuda()
U = torch.empty_like(B)
qy, qx = B.shape
L = nat.lib()
h = cache.reduced(w.op)
out2 = np.zeros(2)
s = nat.stream()


def native():
    nat.check(L.sfb_reduced_solve(h, nat.ptr(B), qx, nat.ptr(U), qx, nat.dptr(out2), s), "reduced")


def native_nosync():
    nat.check(L.sfb_reduced_solve(h, nat.ptr(B), qx, nat.ptr(U), qx, None, s), "reduced")


for _ in range(reps):
    native()
torch.cuda.synchronize()
if reps > 5:
    def t(fn, n=reps):
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / n * 1e3
    print(f"{name} q={qy}")
    print(f"solve_reduced (python, device in) {t(lambda: pb.solve_reduced(w.op, B, cache)):8.3f} ms")
    print(f"sfb_reduced_solve (+ scalar sync) {t(native):8.3f} ms")
    print(f"sfb_reduced_solve (no sync)       {t(native_nosync):8.3f} ms")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        native_nosync()
    e1.record()
    torch.cuda.synchronize()
    print(f"device time per solve (events)    {e0.elapsed_time(e1) / reps:8.3f} ms")
