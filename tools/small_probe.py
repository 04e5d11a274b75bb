"""Tiny MO-PCG (N=32) for launch-overhead analysis under ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_01173_b200 as pb
from paper_2109_01173_b200 import workloads as wl
w = wl.cfg3(N=int(sys.argv[1]) if len(sys.argv) > 1 else 32)
rhs = torch.from_numpy(w.rhs).cuda()
pre = pb.Preconditioner() if (len(sys.argv) > 2 and sys.argv[2] == "identity") else \
    pb.make_preconditioner("elliptic_xnormal", w.x, w.y, mode=sys.argv[2] if len(sys.argv) > 2 else "banded")
for _ in range(3):
    r = pb.mo_pcg(w.op, rhs, precond=pre, stop=pb.relative_residual(1e-30), max_iter=20)
print("ok", r.iterations, r.diagnostics["device"]["loop_ms"])
