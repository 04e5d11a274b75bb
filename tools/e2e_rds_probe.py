"""Where one end-to-end cfg5 IMEX step (numpy states in / out through imex_euler_rds) spends its time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2109_01173_b200 as pb  # noqa: E402
from paper_2109_01173_b200 import _native as nat  # noqa: E402
from paper_2109_01173_b200 import workloads as wl  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8191
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = wl.cfg5(N=N, mode="inverse")
ex = w.extra
p = ex["params"]
inner = pb.InnerSolver(rule="budget", max_iter=K, precond_mode="inverse")
run = dict(domain=pb.SQUARE, x=w.x, y=w.y, d_u=1.0, d_v=p.d_theta, kinetics=ex["kinetics"], rho=p.rho, inner=inner,
           lumped=True)
grid1 = pb.TimeGrid(ex["tau"], ex["tau"])
acc = {}


def timed(name, fn):
    def wrap(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn(*a, **k)
        torch.cuda.synchronize()
        acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
        return out
    return wrap


pinned = [torch.empty(s.shape, dtype=torch.float64, pin_memory=True) for s in ex["state0"]]
for pbuf, s in zip(pinned, ex["state0"]):
    pbuf.copy_(torch.from_numpy(np.ascontiguousarray(s)))
h = tuple(pbuf.numpy() for pbuf in pinned)
for _ in range(3):
    h = pb.imex_euler_rds(state0=h, grid=grid1, **run).final
d = tuple(torch.from_numpy(a).cuda() for a in h)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    d = pb.imex_euler_rds(state0=d, grid=grid1, **run).final
torch.cuda.synchronize()
dev = (time.perf_counter() - t0) / 3
nat.to_device = timed("to_device", nat.to_device)
nat.to_host = timed("to_host", nat.to_host)
L = nat.lib()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    h = pb.imex_euler_rds(state0=h, grid=grid1, **run).final
torch.cuda.synchronize()
e2e = (time.perf_counter() - t0) / 3
for rep in range(2):  # drift check: 10 device-resident steps, 10 numpy steps, twice
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        d = pb.imex_euler_rds(state0=d, grid=grid1, **run).final
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for _ in range(10):
        h = pb.imex_euler_rds(state0=h, grid=grid1, **run).final
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"round {rep}: device-resident {1e2 * (t1 - t0):.1f} ms/step, numpy in/out {1e2 * (t2 - t1):.1f} ms/step", flush=True)
print(f"device-resident step {dev * 1e3:.1f} ms; numpy in/out step {e2e * 1e3:.1f} ms; "
      + ", ".join(f"{k} {v / 3 * 1e3:.1f} ms" for k, v in acc.items()))
