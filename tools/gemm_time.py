"""Live timing of the DMMA GEMM (C = A Bt^T) at q x q x q: python tools/gemm_time.py [q ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2109_01173_b200 import _native as nat  # noqa: E402

L = nat.lib()
s = torch.cuda.current_stream().cuda_stream
for q in [int(a) for a in sys.argv[1:]] or [2047]:
    ld = q + (q % 2)
    A = torch.randn(q, ld, dtype=torch.float64, device="cuda")
    B = torch.randn(q, ld, dtype=torch.float64, device="cuda")
    C = torch.empty(q, ld, dtype=torch.float64, device="cuda")

    def run():
        nat.check(L.sfb_dgemm_nt(A.data_ptr(), ld, B.data_ptr(), ld, q, q, q, C.data_ptr(), ld, s))

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ref = A[:, :q] @ B[:, :q].T
    err = float((C[:, :q] - ref).norm() / ref.norm())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"q={q} {ms * 1e3:8.1f} us  {2 * q ** 3 / ms / 1e9:6.2f} TF/s  rel err vs torch {err:.1e}")
