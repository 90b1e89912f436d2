"""Grouped FP64 tensor-core GEMM (csrc/dgemm.cu) vs cuBLAS DGEMM on the W-build
shapes (P^s X^s: n_s x n_s times n_s x B for every subdomain) and a square
case; correctness (max error relative to cuBLAS) and TFLOP/s of both, CUDA
events on the context stream.
    python profiles/dgemm_bench.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2106_10913_b200 import awg  # noqa: E402

a = awg.SparseSymMatrix(1, np.array([0, 1]), np.array([0]), np.array([1.0]))
ctx = awg.ProblemContext(a, None, awg.Partition([np.array([0])], 1))
cases = {"square_4096": (4096, 4096, 4096, 1), "c2_wpass_B512": (4612, 512, 4612, 16),
         "c5_wpass_B365": (5376, 365, 5376, 216), "ragged_1001x77x333": (1001, 77, 333, 3),
         # W^T (A W): split-K slices of c5's n = 884,736 (C = A^T B)
         "c5_wtaw_TN": (2913, 512, 110592, 8), "square_4096_TN": (4096, 4096, 4096, 1)}
if len(sys.argv) > 1:
    cases = {k: v for k, v in cases.items() if k in sys.argv[1:]}
res = {}
for name, (m, n, k, cnt) in cases.items():
    ta = name.endswith("_TN")
    res[name] = dict(ctx.bench_dgemm(m, n, k, cnt, reps=3, transpose_a=ta), m=m, n=n, k=k, count=cnt, transpose_a=ta)
print(json.dumps(res))
