"""Time the local-solve kernels on synthetic factors at full scale for several
single-pass pipeline settings (env knobs read at context creation).
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
    settings = [("two-pass", {"AWG_NN_TWO_PASS": "1"})]
    mode = os.environ.get("SWEEP", "pipeline")
    if mode == "tasks":  # task granularity and the guided tail, default pipeline
        for mincols, chunks, tail in itertools.product([32, 64, 128, 256], [8, 16, 32], [0, 10, 20]):
            settings.append((f"min{mincols}_chunks{chunks}_tail{tail}",
                             {"AWG_FUSED_MINCOLS": str(mincols), "AWG_FUSED_CHUNKS": str(chunks),
                              "AWG_FUSED_TAIL": str(tail)}))
    elif mode == "static":  # static per-CTA column shares vs the atomic queue, cross-task prefetch
        for st, pf, cpb in itertools.product([0, 1], [0, 1], [0, 1]):
            settings.append((f"static{st}_prefetch{pf}_cpb{cpb or 'auto'}",
                             {"AWG_FUSED_STATIC": str(st), "AWG_FUSED_PREFETCH": str(pf),
                              "AWG_FUSED_CPB": str(cpb)}))
        settings.append(("static0_prefetch1_cpbauto_again", {"AWG_FUSED_STATIC": "0"}))
        settings.append(("static1_prefetch1_cpbauto_again", {"AWG_FUSED_STATIC": "1"}))
    elif mode == "hold":  # column values held in registers across the reduction (AWG_FUSED_HOLD)
        for hold, cpb, nbuf in itertools.product([0, 1], [1, 2], [3, 4, 6]):
            settings.append((f"hold{hold}_cpb{cpb}_nbuf{nbuf}",
                             {"AWG_FUSED_HOLD": str(hold), "AWG_FUSED_CPB": str(cpb), "AWG_FUSED_NBUF": str(nbuf)}))
    else:
        for cpb, nbuf, chunks in itertools.product([1, 2], [2, 3, 4], [4, 8, 16]):
            settings.append((f"cpb{cpb}_nbuf{nbuf}_chunks{chunks}",
                             {"AWG_FUSED_CPB": str(cpb), "AWG_FUSED_NBUF": str(nbuf),
                              "AWG_FUSED_CHUNKS": str(chunks)}))
    for name, env in settings:
        for k in ("AWG_NN_TWO_PASS", "AWG_FUSED_CPB", "AWG_FUSED_NBUF", "AWG_FUSED_CHUNKS", "AWG_FUSED_MINCOLS",
                  "AWG_FUSED_TAIL", "AWG_FUSED_HOLD", "AWG_FUSED_STATIC", "AWG_FUSED_PREFETCH"):
            os.environ.pop(k, None)
        os.environ.update(env)
        try:
            ctx = awg.context_from_problem(p)
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
            rows.append({"setting": name, "error": str(e)[:120]})
    rows.sort(key=lambda r: r.get("h1_ms", 1e9))
    print(json.dumps({"config": cfg, "results": rows}))
