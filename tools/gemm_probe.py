"""Standalone launches of the DMMA GEMM and the banded operator kernel for ncu
(no graphs).  python tools/gemm_probe.py [q] [reps]"""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import numpy as np
from paper_2109_01173_b200 import _native as nat
from paper_2109_01173_b200 import workloads as wl

q = int(sys.argv[1]) if len(sys.argv) > 1 else 2047
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
L = nat.lib()
ld = q + (q % 2)
A = torch.randn(q, ld, dtype=torch.float64, device="cuda")
B = torch.randn(q, ld, dtype=torch.float64, device="cuda")
C = torch.empty(q, ld, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    nat.check(L.sfb_dgemm_nt(A.data_ptr(), ld, B.data_ptr(), ld, q, q, q, C.data_ptr(), ld, s))
ref = A[:, :q] @ B[:, :q].T
err = float((C[:, :q] - ref).norm() / ref.norm())
w = wl.cfg3(N=(q + 2) // 2 * 2)
U = torch.randn(w.op.shape, dtype=torch.float64, device="cuda")
for _ in range(reps):
    W = w.op.apply(U)
torch.cuda.synchronize()
print(f"q={q} gemm rel err vs cuBLAS {err:.2e}")
