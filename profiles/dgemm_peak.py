"""FP64 DGEMM throughput on this B200 (cuBLAS via torch.matmul, CUDA events):
the square peak and the W-build shapes (P^s X with n_s x n_s times n_s x B).
MEASURED_PEAKS.json has no fp64 entry; the W-build roofline uses this.
    python profiles/dgemm_peak.py"""
import json

import torch

res = {}
for name, (m, k, n) in {"square_8192": (8192, 8192, 8192), "wbuild_c5_B365": (5376, 5376, 365),
                        "wbuild_c5_B512": (5376, 5376, 512), "wbuild_c2_B512": (4612, 4612, 512)}.items():
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[name] = {"ms": ms, "tflops": 2.0 * m * k * n / ms / 1e9}
print(json.dumps(res))
