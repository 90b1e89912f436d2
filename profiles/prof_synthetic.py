"""ncu target: the dominant solve kernels at a config's full scale on synthetic
factors (V^s hash-filled with the config's subdomain sizes, W with n_minus
columns), no setup.  The profiler range covers one launch of each:
single-pass local solve, W^T x, W c, SpMV.
    ncu --profile-from-start off --set full ... python profiles/prof_synthetic.py c5 2913"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_10913_b200 import awg, problems  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
p = problems.make(cfg)
nm = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ctx = awg.context_from_problem(p, options={"synth_nm": nm})
ctx.synthetic_factors(m_per_sub=8)
names = ["nn_fused", "spmv"] + (["w_gemvT", "w_gemv"] if nm else [])
for name in names:  # warm-up (module load, first-launch attributes)
    ctx.time_kernel(name, reps=1)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for name in names:
    ctx.time_kernel(name, reps=1)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
ctx.close()
print("ok", cfg, names)
