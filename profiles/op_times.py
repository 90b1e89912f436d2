"""Device time of each operator of the H3 apply (awg_time_apply: the op run
back to back on device buffers, CUDA events on the library stream), to see
where a PCG iteration goes beyond the local solve.
    python profiles/op_times.py [config]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_10913_b200 import awg, problems  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
p = problems.make(cfg)
ctx = awg.context_from_problem(p)
ctx.setup(awg.config_for(p))
x, rep = ctx.pcg(p.b, p.rtol, 10000)
out = {"config": cfg, "iterations": rep.iterations, "ms_per_iteration": rep.solve_ms / max(rep.iterations, 1)}
for name in ("A", "AMINUS", "APLUS", "H1", "Q", "QW", "H2", "H3"):
    out[name] = ctx.time_apply(getattr(awg.Op, name), reps=20)
for k in ("nn_fused", "spmv", "w_gemvT", "w_gemv"):
    out["kernel_" + k] = ctx.time_kernel(k, reps=10)[0]
print(json.dumps(out))
