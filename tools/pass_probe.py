"""Per-pass device time of one MO-PCG iteration (cfg3 operator).

    python tools/pass_probe.py [N] [mode]

Runs a few identity-preconditioned iterations to populate the solver, then
times the banded operator pass and the vector update pass back to back and
prints algorithmic GB/s (32 q^2 and 48 q^2 bytes).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2109_01173_b200 as pb  # noqa: E402
from paper_2109_01173_b200 import workloads as wl  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
mode = sys.argv[2] if len(sys.argv) > 2 else "identity"
w = wl.cfg3(N=N)
qy, qx = w.op.shape
rhs = torch.from_numpy(w.rhs).cuda()
pre = pb.Preconditioner() if mode == "identity" else pb.make_preconditioner("elliptic_xnormal", w.x, w.y, mode=mode)
pb.mo_pcg(w.op, rhs, precond=pre, stop=pb.relative_residual(1e-30), max_iter=5)
t = pb.solvers.pcg_pass_times(w.op, pre, reps=30)
n2 = qy * qx * 8
print(f"N={N} operator pass {t['operator_ms'] * 1e3:7.1f} us {4 * n2 / t['operator_ms'] / 1e6:7.0f} GB/s | "
      f"update {t['update_ms'] * 1e3:7.1f} us {6 * n2 / t['update_ms'] / 1e6:7.0f} GB/s | "
      f"precond ({mode}) {t['preconditioner_ms'] * 1e3:7.1f} us")
