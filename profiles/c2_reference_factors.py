"""The exported-factor protocol at BASELINE config c2 with
THE REFERENCE'S OWN FACTORS: the replay of oracle/run_memo_reference.sh exports
every setup product of the reference (V^s, lambda, Y, K0, W, KW: 2.9 GB, too
large to commit) and its applies of every operator on three seeded vectors and
its PCG solve.  The device loads those factors (awg_load_factors) and must
reproduce the applies within 1e-11 (A bit-identical) and the solve within +-1
iteration / 1e-7.  One-off run (the factors travel with the gpurun snapshot
from scratch space); the log is committed under profiles/.
    python profiles/c2_reference_factors.py <dir with the replay's out/*.npy> <reference|exact>"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_10913_b200 import awg, problems  # noqa: E402

d, sem = sys.argv[1], sys.argv[2]
g = {f[:-4]: np.load(os.path.join(d, f)) for f in os.listdir(d) if f.endswith(".npy") and f not in ("v_minus.npy",)}
with open(os.path.join(d, "summary.json")) as fh:
    s = json.load(fh)
p = problems.make("c2")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def ctx_for(mode):
    cfg = awg.config_for(p, rrf_semantics=sem)
    cfg.awg = mode
    c = awg.context_from_problem(p)
    c.load_factors(cfg, g)
    return c


OPS = {"A": awg.Op.A, "Aminus": awg.Op.AMINUS, "Aplus": awg.Op.APLUS, "H1": awg.Op.H1, "Q": awg.Op.Q, "QW": awg.Op.QW,
       "H2": awg.Op.H2, "PI3": awg.Op.PI3, "PI3T": awg.Op.PI3T}
out = {"semantics": sem, "n0": s["n0"], "r0": s["r0"], "n_minus": s["n_minus"], "rw": s["rw"], "applies": {}}
ctx = ctx_for(awg.AwgMode.AD)
for name, op in OPS.items():
    e = 0.0
    for x, y in zip(g["x_apply"], g["y_" + name]):
        got = ctx.apply(op, x)
        e = max(e, 0.0 if np.array_equal(got, y) else rel(got, y))
    out["applies"][name] = e
for mode, key in ((awg.AwgMode.AD, "H3ad"), (awg.AwgMode.HYB, "H3hyb"), (awg.AwgMode.INEX, "H3inex")):
    c = ctx if mode == awg.AwgMode.AD else ctx_for(mode)
    got = [c.apply(awg.Op.H3, x) for x in g["x_apply"]]
    if key == "H3inex" and not np.isfinite(g["y_" + key]).all():
        # the reference's lu_solve (bug 2, dense.cpp:404-409) overflows on c2's INEX core:
        # its own output is not finite; the bug-compatible device path must not be finite either
        out["applies"][key] = {"reference_nonfinite": int((~np.isfinite(g["y_" + key])).sum()),
                               "device_nonfinite": int(sum((~np.isfinite(y)).sum() for y in got))}
    else:
        out["applies"][key] = max(rel(a, y) for a, y in zip(got, g["y_" + key]))
    if c is not ctx:
        c.close()
# INEX with the exact LU solve against the restatement on the same (reference) factors
from oracle import awg_oracle as O  # noqa: E402  (checker only)

orc = O.AwgOracle(p.n, p.row_offsets, p.col_indices, p.values, list(p.omega), g)
orc.lu_exact = True
cfg = awg.config_for(p, rrf_semantics=sem, lu_semantics="exact")
cfg.awg = awg.AwgMode.INEX
ci = awg.context_from_problem(p)
ci.load_factors(cfg, g)
out["applies"]["H3inex_exact_lu_vs_restatement"] = max(rel(ci.apply(awg.Op.H3, x), orc.h3(x, "inex"))
                                                       for x in g["x_apply"][:2])
ci.close()
x, rep = ctx.pcg(p.b, p.rtol, 10 * p.n)
k = min(len(rep.residual_history), len(g["pcg_residuals"]))
rh, rg = np.asarray(rep.residual_history[:k]), np.asarray(g["pcg_residuals"][:k])
out["pcg"] = {"iterations": rep.iterations, "reference_iterations": s["iterations"], "x_rel": rel(x, g["pcg_x"]),
              "kappa": rep.kappa_estimate, "reference_kappa": s["kappa"],
              "residual_history_max_reldiff": float(np.max(np.abs(rh - rg) / rg)),
              "solve_ms": rep.solve_ms, "reference_t_solve_s": s["t_solve"]}
ms = ctx.time_apply(awg.Op.H3, 20) if hasattr(ctx, "time_apply") else None
out["h3_apply_ms"] = ms
out["reference_t_h3_apply_s"] = s["t_h3_apply"]
print(json.dumps(out))
