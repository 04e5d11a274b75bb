"""Live timing of the batched DMMA GEMM (nb products of h^3 in one persistent launch):
python tools/batch_gemm_time.py [nb h ...]   (default: 343 1024, the cfg5 Strassen leaves)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2109_01173_b200 import _native as nat  # noqa: E402

L = nat.lib()
s = torch.cuda.current_stream().cuda_stream
args = [int(a) for a in sys.argv[1:]] or [343, 1024]
for nb, h in zip(args[0::2], args[1::2]):
    A = torch.randn(nb, h, h, dtype=torch.float64, device="cuda")
    B = torch.randn(nb, h, h, dtype=torch.float64, device="cuda")
    out = torch.empty(nb, h, h, dtype=torch.float64, device="cuda")

    def run():
        nat.check(L.sfb_dgemm_nt_batch(nb, A.data_ptr(), h, B.data_ptr(), h, h, h, h, out.data_ptr(), h, h * h, s))

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    err = max(float((out[b] - A[b] @ B[b].T).norm() / (A[b] @ B[b].T).norm()) for b in (0, nb - 1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{nb} x {h}^3: {ms * 1e3:9.1f} us  {2 * nb * h ** 3 / ms / 1e9:6.2f} TF/s  rel err vs torch {err:.1e}")
