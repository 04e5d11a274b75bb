"""Where the time of a small reduced solve (cfg1, q = 256) goes.

    python tools/reduced_probe.py [cfg1|cfg2]
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

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
w = wl.CONFIGS[name]()
cache = pb.build_spectral_cache(w.op)
cache.native()
B = torch.from_numpy(w.rhs).cuda()
U = torch.empty_like(B)
qy, qx = B.shape
L = nat.lib()


def t(fn, reps=200):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


out2 = np.zeros(2)
print(f"{name} q={qy}")
print(f"solve_reduced (device in)  {t(lambda: pb.solve_reduced(w.op, B, cache)):8.3f} ms")
print(f"sfb_pre_apply              {t(lambda: L.sfb_pre_apply(cache.native(), nat.ptr(B), qx, nat.ptr(U), qx, nat.stream())):8.3f} ms")
print(f"sfb_op_residual            {t(lambda: L.sfb_op_residual(w.op.native(), nat.ptr(U), qx, nat.ptr(B), qx, nat.dptr(out2), nat.stream())):8.3f} ms")
print(f"check_pencils              {t(lambda: cache.check_pencils()):8.3f} ms")
print(f"empty_like                 {t(lambda: torch.empty_like(B)):8.3f} ms")
