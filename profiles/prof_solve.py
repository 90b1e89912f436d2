"""Profiling driver: GPU setup (not profiled), then ONE PCG solve bracketed by
cudaProfilerStart/Stop so `ncu --profile-from-start off` sees only the hot
path.  python profiles/prof_solve.py <config> [rrf]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2106_10913_b200 import awg, problems  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
p = problems.make(cfg_name)
ctx = awg.context_from_problem(p)
ctx.setup(awg.config_for(p, rrf_semantics=sys.argv[2] if len(sys.argv) > 2 else "reference"))
x, rep = ctx.pcg(p.b, p.rtol, 10000)  # warm (graph capture, lazy module loads)
torch.cuda.synchronize()
torch.cuda.profiler.start()
x, rep = ctx.pcg(p.b, p.rtol, 10000)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"{cfg_name}: {rep.iterations} iterations, {rep.solve_ms:.2f} ms")
