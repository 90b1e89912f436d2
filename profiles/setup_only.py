"""GPU setup only (phase timings on stderr: option verbose=1/2 from VERBOSE).
    python profiles/setup_only.py <config> [rrf]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_10913_b200 import awg, problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
p = problems.make(name)
ctx = awg.context_from_problem(p, options={"verbose": int(os.environ.get("VERBOSE", "1"))})
t = time.time()
ctx.setup(awg.config_for(p, rrf_semantics=sys.argv[2] if len(sys.argv) > 2 else "reference"))
q = ctx.query()
print(json.dumps({"config": name, "setup_s": time.time() - t, "n0": q["n0"], "n_minus": q["n_minus"],
                  "w_inner_total": q.get("w_inner_total"), "w_block_passes": q.get("w_batches"),
                  "t_setup_ms": q.get("t_setup_ms")}))
