"""Per-iteration device time of MO-PCG for several preconditioner forms.

    python tools/iter_probe.py [N] [iters]

Prints ms/iteration (device loop time of the CUDA-graph loop) for the
identity, banded and inverse preconditioners on the cfg3 operator; the
identity run isolates the operator + vector passes of an iteration.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2109_01173_b200 as pb  # noqa: E402
from paper_2109_01173_b200 import workloads as wl  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
its = int(sys.argv[2]) if len(sys.argv) > 2 else 100
w = wl.cfg3(N=N)
rhs = torch.from_numpy(w.rhs).cuda()
stop = pb.relative_residual(1e-30)
for name in ("identity", "banded", "inverse"):
    pre = pb.Preconditioner() if name == "identity" else \
        pb.make_preconditioner("elliptic_xnormal", w.x, w.y, mode=name)
    for _ in range(2):
        pb.mo_pcg(w.op, rhs, precond=pre, stop=stop, max_iter=its)
    r = pb.mo_pcg(w.op, rhs, precond=pre, stop=stop, max_iter=its)
    ms = r.diagnostics["device"]["loop_ms"]
    print(f"N={N} {name:9s} {ms / its * 1e3:8.1f} us/iteration ({its} iterations)")
