"""Profiling driver: GPU setup (not profiled), then ONE PCG solve bracketed by
cudaProfilerStart/Stop so `ncu --profile-from-start off` sees only the hot
path.
    python profiles/prof_solve.py <config> [rrf] [w_rtol]

w_rtol (default: the reference's 1e-10): gpurun only starts ncu after the same
command ran to completion without it in under 300 s, and the c5 setup alone is
~315 s (255 s of it the W inner PCGs).  With w_rtol = 1e-2 the inner PCGs stop
after a few iterations: V^s, lambda, Z, K0 are the real c5 factors, W and KW
have the real shapes (n x n_minus, rw x rw) but W's columns are only roughly
solved.  Every solve-phase kernel then runs on the same shapes and the same
local factors as in the bench; only the PCG's iteration count differs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2106_10913_b200 import awg, problems  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
rrf = sys.argv[2] if len(sys.argv) > 2 else "reference"
kw = {"rrf_semantics": rrf}
if len(sys.argv) > 3:
    kw["w_rtol"] = float(sys.argv[3])
p = problems.make(cfg_name)
ctx = awg.context_from_problem(p)
ctx.setup(awg.config_for(p, **kw))
x, rep = ctx.pcg(p.b, p.rtol, 10000)  # warm (graph capture, lazy module loads)
torch.cuda.synchronize()
torch.cuda.profiler.start()
x, rep = ctx.pcg(p.b, p.rtol, 10000)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
q = ctx.query()
print(f"{cfg_name}: {rep.iterations} iterations, {rep.solve_ms:.2f} ms, converged {rep.converged}, "
      f"n0 {q['n0']}, n_minus {q['n_minus']}, rw {q.get('rw')}, setup {q.get('t_setup_ms')}")
