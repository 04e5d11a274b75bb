"""In-loop time of the banded sandwich kernel on aligned (padded) grids.

    python tools/band_probe.py [N]

Times sfb_op_apply (plain loader, 5 terms) back to back with CUDA events on
padded device buffers (no staging copy), and reports algorithmic GB/s
(one read of U + one write of W per launch).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2109_01173_b200 import _native as nat  # noqa: E402
from paper_2109_01173_b200 import workloads as wl  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
w = wl.cfg3(N=N)
qy, qx = w.op.shape
ld = (qx + 31) // 32 * 32
L = nat.lib()
s = torch.cuda.current_stream().cuda_stream
U = torch.randn(qy, ld, dtype=torch.float64, device="cuda")
W = torch.empty_like(U)
h = w.op.native()


def run():
    L.sfb_op_apply(h, U.data_ptr(), ld, W.data_ptr(), ld, s)


for _ in range(5):
    run()
torch.cuda.synchronize()
reps = 100
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / reps * 1e3
gbs = 2 * qy * qx * 8 / (us * 1e-6) / 1e9
print(f"N={N} band kernel (plain, {len(w.op.terms)} terms) {us:7.1f} us  {gbs:7.0f} GB/s algorithmic")
