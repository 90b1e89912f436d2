"""Per-iteration device time of the c2 solve (op_times-style) under knob
settings given as NAME=VALUE[,NAME=VALUE] arguments (awg_set_option names),
one fresh context each.
    python profiles/knob_sweep.py c2 "pdl_early=0" "pdl_early=1,rows_group=8" ..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_10913_b200 import awg, problems  # noqa: E402

cfg = sys.argv[1]
p = problems.make(cfg)
out = []
for spec in sys.argv[2:]:
    opts = {k: int(v) for k, v in (kv.split("=") for kv in spec.split(",") if kv)}
    try:
        ctx = awg.context_from_problem(p, options=opts)
        kind = os.environ.get("ONE_LEVEL", "NN")  # NN | AS | AS_PLUS
        ctx.setup(awg.config_for(p, one_level=getattr(awg.OneLevelKind, kind)))
        best = 1e9
        x, rep = ctx.pcg(p.b, p.rtol, 10000)
        ctx.kernel_timer(reset=True)
        for _ in range(3):
            x, rep = ctx.pcg(p.b, p.rtol, 10000)
            best = min(best, rep.solve_ms / max(rep.iterations, 1))
        kms, kl = ctx.kernel_timer()
        out.append({"knobs": spec, "iterations": rep.iterations, "ms_per_iteration": best,
                    "local_solve_ms_in_solve": kms / max(kl, 1), "H1_ms": ctx.time_apply(awg.Op.H1, reps=20),
                    "H3_ms": ctx.time_apply(awg.Op.H3, reps=20), "Q_ms": ctx.time_apply(awg.Op.Q, reps=20),
                    "APLUS_ms": ctx.time_apply(awg.Op.APLUS, reps=20)})
        ctx.close()
    finally:
        pass
print(json.dumps({"config": cfg, "results": out}))
