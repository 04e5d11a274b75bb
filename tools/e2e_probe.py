"""Where the end-to-end (numpy in / numpy out) time of a cfg3 MO-PCG solve goes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2109_01173_b200 as pb  # noqa: E402
from paper_2109_01173_b200 import _native as nat  # noqa: E402
from paper_2109_01173_b200 import workloads as wl  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
w = wl.cfg3(N=N)
stop = pb.relative_residual(1e-30)


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


pinned_rhs = torch.empty(w.rhs.shape, dtype=torch.float64, pin_memory=True)
pinned_rhs.copy_(torch.from_numpy(w.rhs))
rhs = pinned_rhs.numpy() if os.environ.get("E2E_PINNED", "1") == "1" else w.rhs  # bench.py's e2e input is pinned
d = nat.to_device(rhs)
print(f"to_device (numpy H2D)    {t(lambda: nat.to_device(rhs)):7.2f} ms")
print(f"cpu().numpy() (D2H)      {t(lambda: d.cpu().numpy()):7.2f} ms")
pin = torch.empty(d.shape, dtype=torch.float64, pin_memory=True)
pin2 = torch.empty_like(pin).pin_memory(); d2 = torch.empty_like(d)
print(f"pinned H2D               {t(lambda: d2.copy_(pin2, non_blocking=True)):7.2f} ms")
print(f"pinned D2H               {t(lambda: pin.copy_(d, non_blocking=True)):7.2f} ms")
print(f"numpy -> pinned memcpy   {t(lambda: pin.numpy().__setitem__(Ellipsis, rhs)):7.2f} ms")
pre = w.precond
for it in (0, 50):
    print(f"mo_pcg device  {it:3d} it  {t(lambda: pb.mo_pcg(w.op, d, precond=pre, stop=stop, max_iter=it), 3):8.2f} ms")
    print(f"mo_pcg numpy   {it:3d} it  {t(lambda: pb.mo_pcg(w.op, rhs, precond=pre, stop=stop, max_iter=it), 3):8.2f} ms")
r = pb.mo_pcg(w.op, d, precond=pre, stop=stop, max_iter=50)
print("device run:", r.iterations, r.stop_reason, r.diagnostics["device"])
r = pb.mo_pcg(w.op, rhs, precond=pre, stop=stop, max_iter=50)
print("numpy run:", r.iterations, r.stop_reason, r.diagnostics["device"])
# the bench's e2e loop, verbatim
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(2):
    torch.cuda.synchronize()
    e0.record()
    w0 = time.perf_counter()
    its_e = 0
    for _ in range(3):
        rh = pb.mo_pcg(w.op, rhs, precond=pre, stop=stop, max_iter=50)
        its_e += rh.iterations
    e1.record()
    torch.cuda.synchronize()
    el = e0.elapsed_time(e1)
    print(f"bench-style e2e: {el / 3:.2f} ms/step (events), {(time.perf_counter() - w0) * 1e3 / 3:.2f} ms/step (wall)")
# phase breakdown of the numpy path
for rep in range(4):
    torch.cuda.synchronize()
    a = time.perf_counter()
    B = nat.to_device(rhs)
    torch.cuda.synchronize()
    b = time.perf_counter()
    rr = pb.mo_pcg(w.op, B, precond=pre, stop=stop, max_iter=50)
    torch.cuda.synchronize()
    c = time.perf_counter()
    Uh = rr.solution.cpu().numpy()
    d_ = time.perf_counter()
    print(f"phases: H2D {1e3*(b-a):.2f}  solve {1e3*(c-b):.2f} (loop {rr.diagnostics['device']['loop_ms']:.2f})  D2H {1e3*(d_-c):.2f} ms")
