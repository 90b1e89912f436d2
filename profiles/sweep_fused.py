"""Time the local-solve kernels on synthetic factors at full scale for several
single-pass pipeline settings (awg_set_option switches).
    python profiles/sweep_fused.py c2 c5"""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_10913_b200 import awg, problems  # noqa: E402

for cfg in sys.argv[1:] or ["c2"]:
    p = problems.make(cfg)
    rows = []
    settings = [("two-pass", {"nn_two_pass": 1})]
    mode = os.environ.get("SWEEP", "pipeline")
    if mode == "tasks":  # task granularity and the guided tail, default pipeline
        for mincols, chunks, tail in itertools.product([32, 64, 128, 256], [8, 16, 32], [0, 10, 20]):
            settings.append((f"min{mincols}_chunks{chunks}_tail{tail}",
                             {"fused_min_cols": mincols, "fused_chunks": chunks,
                              "fused_tail": tail}))
    elif mode == "static":  # static per-CTA column shares vs the atomic queue, cross-task prefetch
        for st, pf, cpb in itertools.product([0, 1], [0, 1], [0, 1]):
            settings.append((f"static{st}_prefetch{pf}_cpb{cpb or 'auto'}",
                             {"fused_static": st, "fused_prefetch": pf,
                              "fused_cpb": cpb}))
        settings.append(("static0_prefetch1_cpbauto_again", {"fused_static": 0}))
        settings.append(("static1_prefetch1_cpbauto_again", {"fused_static": 1}))
    elif mode == "hold":  # column values held in registers across the reduction (option fused_hold)
        for hold, cpb, nbuf in itertools.product([0, 1], [1, 2], [3, 4, 6]):
            settings.append((f"hold{hold}_cpb{cpb}_nbuf{nbuf}",
                             {"fused_hold": hold, "fused_cpb": cpb, "fused_nbuf": nbuf}))
    else:
        for cpb, nbuf, chunks in itertools.product([1, 2], [2, 3, 4], [4, 8, 16]):
            settings.append((f"cpb{cpb}_nbuf{nbuf}_chunks{chunks}",
                             {"fused_cpb": cpb, "fused_nbuf": nbuf,
                              "fused_chunks": chunks}))
    for name, env in settings:
        try:
            ctx = awg.context_from_problem(p, options=env)
            ctx.synthetic_factors(m_per_sub=8)
            if name == "two-pass":
                a = ctx.time_kernel("nn_gemvT", reps=5)
                b = ctx.time_kernel("nn_gemv", reps=5)
                ms, by = a[0] + b[0], a[1] + b[1]
            else:
                ms, by = ctx.time_kernel("nn_fused", reps=5)
            h1 = ctx.time_apply(awg.Op.H1, reps=5)
            rows.append({"setting": name, "kernel_ms": ms, "GBps": by / ms / 1e6, "h1_ms": h1})
            ctx.close()
        except Exception as e:  # noqa: BLE001
            rows.append({"setting": name, "error": e[:120]})
    rows.sort(key=lambda r: r.get("h1_ms", 1e9))
    print(json.dumps({"config": cfg, "results": rows}))
