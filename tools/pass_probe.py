"""Per-pass device time of one MO-PCG iteration (cfg3 operator).

    python tools/pass_probe.py [N] [mode]

Runs a few identity-preconditioned iterations to populate the solver, then
times the banded operator pass and the vector update pass back to back and
prints algorithmic GB/s (48 q^2 and 24 q^2 bytes: the operator pass also
carries the previous iteration's deferred U += alpha Q).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2109_01173_b200 as pb  # noqa: E402
from paper_2109_01173_b200 import workloads as wl  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
mode = sys.argv[2] if len(sys.argv) > 2 else "identity"
cfg = sys.argv[3] if len(sys.argv) > 3 else "cfg3"  # cfg3 (P2, 5 terms) or cfg4 (P4 heat step, 5 terms)
w = wl.CONFIGS[cfg](N=N)
qy, qx = w.op.shape
rhs = torch.from_numpy(w.rhs if w.rhs is not None else
                       np.random.default_rng(0).standard_normal(w.op.shape)).cuda()
if mode == "identity":
    pre = pb.Preconditioner()
elif cfg == "cfg3":
    pre = pb.make_preconditioner("elliptic_xnormal", w.x, w.y, mode=mode)
else:
    pre = pb.make_preconditioner("parabolic", w.x, w.y, d_u=1.0, tau=1e-3, mode=mode)
pb.mo_pcg(w.op, rhs, precond=pre, stop=pb.relative_residual(1e-30), max_iter=5)
t = pb.solvers.pcg_pass_times(w.op, pre, reps=30)
n2 = qy * qx * 8
print(f"{cfg} N={N} operator pass {t['operator_ms'] * 1e3:7.1f} us {6 * n2 / t['operator_ms'] / 1e6:7.0f} GB/s | "
      f"update {t['update_ms'] * 1e3:7.1f} us {3 * n2 / t['update_ms'] / 1e6:7.0f} GB/s | "
      f"precond ({mode}) {t['preconditioner_ms'] * 1e3:7.1f} us")
