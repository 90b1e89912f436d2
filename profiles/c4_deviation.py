"""c4 under a LABELLED DEVIATION from the reference: w_rtol looser than the
reference's 1e-10 (which build_w's inner PCGs cannot reach on c4-shaped
problems: DESIGN.md §6, profiles/r02e/c4s_reference_w_probe_10n.json).
    python profiles/c4_deviation.py <config> <w_rtol> [rrf]
Prints setup / solve figures; not a bench line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_10913_b200 import awg, problems  # noqa: E402

name, w_rtol = sys.argv[1], float(sys.argv[2])
rrf = sys.argv[3] if len(sys.argv) > 3 else "reference"
p = problems.make(name)
ctx = awg.context_from_problem(p, options={"verbose": 1})
t = time.time()
out = {"config": name, "w_rtol": w_rtol, "rrf": rrf, "deviation": "w_rtol (reference: 1e-10)"}
try:
    ctx.setup(awg.config_for(p, rrf_semantics=rrf, w_rtol=w_rtol))
    q = ctx.query()
    out.update(setup_s=time.time() - t, n0=q["n0"], n_minus=q["n_minus"], rw=q.get("rw"),
               w_inner_total=q.get("w_inner_total"), w_block_passes=q.get("w_batches"))
    x, rep = ctx.pcg(p.b, p.rtol, 10000)
    out.update(iterations=rep.iterations, converged=bool(rep.converged), final_relres=rep.final_relative_residual,
               solve_ms=rep.solve_ms, kappa=rep.kappa_estimate)
except Exception as e:  # the reference's own outcomes: non-convergence, breakdown
    out.update(error=repr(e), setup_s=time.time() - t)
print(json.dumps(out))
