"""Back-to-back applications of the banded (SPIKE) preconditioner through sfb_pre_apply, for ncu and timing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_01173_b200 as pb
from paper_2109_01173_b200 import _native as nat
from paper_2109_01173_b200 import workloads as wl
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = wl.cfg3(N=N)
qy, qx = w.op.shape
pre = pb.make_preconditioner("elliptic_xnormal", w.x, w.y, mode="banded")
ph = pre.native(w.op.shape)
U = torch.randn(qy, qx, dtype=torch.float64, device="cuda")
Z = torch.empty_like(U)
s = torch.cuda.current_stream().cuda_stream
L = nat.lib()
for _ in range(reps):
    nat.check(L.sfb_pre_apply(ph, U.data_ptr(), qx, Z.data_ptr(), qx, s))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    L.sfb_pre_apply(ph, U.data_ptr(), qx, Z.data_ptr(), qx, s)
e1.record(); torch.cuda.synchronize()
print(f"N={N} banded preconditioner apply {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
