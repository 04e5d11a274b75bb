import time, torch, numpy as np
n = 8192 * 8192
p = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
gb = n * 8 / 1e9
print("H2D pinned tensor      %.1f GB/s" % (gb / t(lambda: d.copy_(p, non_blocking=True))))
print("D2H pinned tensor      %.1f GB/s" % (gb / t(lambda: p.copy_(d, non_blocking=True))))
v = torch.from_numpy(p.numpy())  # numpy view of the pinned block, as the e2e path sees it
print("view is_pinned:", v.is_pinned())
print("H2D numpy view .to()   %.1f GB/s" % (gb / t(lambda: v.to("cuda"))))
def d2h_new():
    o = torch.empty(n, dtype=torch.float64, pin_memory=True); o.copy_(d); return o.numpy()
print("D2H fresh pinned block %.1f GB/s" % (gb / t(d2h_new)))
