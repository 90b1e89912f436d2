"""Time the second-coarse-space kernels (W^T x split-K + column sum, W c) at
full scale on a synthetic W (option synth_nm columns, hash-filled), next to the
single-pass local solve on synthetic factors — no setup needed.
    python profiles/w_kernels.py c3:2105 c5:2913"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_10913_b200 import awg, problems  # noqa: E402

out = []
for spec in sys.argv[1:] or ["c5:2913"]:
    cfg, nm = spec.split(":")
    p = problems.make(cfg)
    ctx = awg.context_from_problem(p, options={"synth_nm": int(nm)})
    ctx.synthetic_factors(m_per_sub=8)
    row = {"config": cfg, "n": p.n, "n_minus": int(nm)}
    for name in ("w_gemvT", "w_gemv", "nn_fused", "spmv"):
        ms, by = ctx.time_kernel(name, reps=5)
        row[name] = {"ms": ms, "GBps": by / ms / 1e6}
    out.append(row)
    ctx.close()
print(json.dumps(out))
