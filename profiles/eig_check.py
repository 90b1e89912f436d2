"""The setup's batched symmetric eigensolver (csrc/eig.cu) on seeded matrices
against cuSOLVER Dsyevd: accuracy and batch timings.
    python profiles/eig_check.py [n:count:kind ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_10913_b200 import awg  # noqa: E402

VERBOSE = int(os.environ.get("VERBOSE", "1"))
specs = sys.argv[1:] or ["300:4:0", "289:2:1", "1024:4:2", "5376:16:0", "5376:148:0"]
for spec in specs:
    n, cnt, kind = (int(v) for v in spec.split(":"))
    opts = {k: int(v) for k, v in (kv.split("=") for kv in os.environ.get("EIG_OPTIONS", "").split(",") if kv)}
    r = awg.bench_eig(n, cnt, kind, verbose=VERBOSE, options=opts)
    print(json.dumps({"n": n, "count": cnt, "kind": kind, **r}), flush=True)
