"""Inverse-form preconditioner apply Z = A R B^T at q x q (two dense products):
classic DMMA GEMMs vs one level of Strassen around them -- time and error
against torch's fp64 matmul.  python tools/strassen_probe.py [q ...]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_01173_b200 import _native as nat  # noqa: E402

L = nat.lib()
s = torch.cuda.current_stream().cuda_stream
PRE_INVERSE = nat.PRE_INVERSE


SPECTRAL = os.environ.get("STRASSEN_PROBE_KIND") == "spectral"  # the 4-product sandwich V_L [(V_L^T R V_R) o K] V_R^T


def make(q, A, Bt, levels):
    prev, prev_l = L.sfb_set_strassen_min_q(256 if levels else 0), L.sfb_set_strassen_levels(levels)
    out = C.c_void_p()
    if SPECTRAL:
        lam = np.linspace(1.0, 2.0, q)
        nat.check(L.sfb_pre_create(q, q, nat.PRE_SPECTRAL_PROD, A.data_ptr(), Bt.data_ptr(), nat.host_ptr(lam),
                                   nat.host_ptr(lam), C.byref(out)), "pre")
    else:
        nat.check(L.sfb_pre_create(q, q, PRE_INVERSE, A.data_ptr(), Bt.data_ptr(), None, None, C.byref(out)), "pre")
    L.sfb_set_strassen_min_q(prev)
    L.sfb_set_strassen_levels(prev_l)
    return out


for q in [int(a) for a in sys.argv[1:]] or [4096, 8192]:
    g = torch.Generator(device="cuda").manual_seed(q)
    A = torch.randn(q, q, dtype=torch.float64, device="cuda", generator=g)
    Bt = torch.randn(q, q, dtype=torch.float64, device="cuda", generator=g)
    R = torch.randn(q, q, dtype=torch.float64, device="cuda", generator=g)
    Z = torch.empty_like(R)
    if SPECTRAL:
        il = 1.0 / torch.linspace(1.0, 2.0, q, dtype=torch.float64, device="cuda")
        ref = A @ ((A.T @ R @ Bt) * (il[:, None] * il[None, :])) @ Bt.T
    else:
        ref = A @ (R @ Bt.T)
    only = os.environ.get("STRASSEN_PROBE_LEVELS")  # e.g. "3": just that schedule (ncu captures)
    for name, levels in (("classic", 0), ("strassen-1", 1), ("strassen-2", 2), ("strassen-3", 3)):
        if only is not None and str(levels) not in only.split(","):
            continue
        h = make(q, A, Bt, levels)
        if L.sfb_pre_uses_strassen(h) != levels:  # leaves below the minimum size
            nat.check(L.sfb_pre_destroy(h), "destroy")
            continue

        def run():
            nat.check(L.sfb_pre_apply(h, R.data_ptr(), q, Z.data_ptr(), q, s), "apply")

        for _ in range(2):
            run()
        torch.cuda.synchronize()
        err = float((Z - ref).norm() / ref.norm())
        emax = float((Z - ref).abs().max() / ref.abs().max())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        nprod = 4 if SPECTRAL else 2
        print(f"q={q} {name:10s} {ms:8.3f} ms per apply ({nprod} products + 2 copies)  "
              f"{2 * nprod * q ** 3 / ms / 1e9:6.2f} TF/s algorithmic  rel err {err:.2e}  max err / max {emax:.2e}", flush=True)
        nat.check(L.sfb_pre_destroy(h), "destroy")
