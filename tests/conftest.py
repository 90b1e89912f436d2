import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


def load_golden(case):
    g = np.load(os.path.join(GOLDEN, case + ".npz"))
    with open(os.path.join(GOLDEN, case + ".json")) as fh:
        s = json.load(fh)
    return g, s


def golden_with_base(case):
    """Variant fixtures (*_exact, *_additive, *_none) store only what differs
    from their base case."""
    g, s = load_golden(case)
    d = {k: g[k] for k in g.files}
    if s.get("base"):
        base, _ = load_golden(s["base"])
        for k in ("V", "Y", "lam", "pencil_lam"):  # what make_golden.py drops from variants
            if k not in d:
                d[k] = base[k]
    return d, s


ALL_CASES = ["c1", "c1_exact", "t2d", "t2d_exact", "t2d_additive", "t2d_ov2", "t3d", "t3d_none", "t3d_blocks",
             "telas", "telas8", "tragged", "t1box"]


def case_options(s):
    """(composition, awg mode) the fixture was generated with (ref_driver args)."""
    args = s.get("args") or []
    comp = args[args.index("--comp") + 1] if "--comp" in args else "hybrid"
    mode = args[args.index("--awg") + 1] if "--awg" in args else "ad"
    return comp, mode


def one_level_of(s):
    args = s.get("args") or []
    return args[args.index("--one-level") + 1] if "--one-level" in args else "NN"


def omega_of(g):
    off, idx = g["part_offsets"], g["part_indices"]
    return [idx[a:b] for a, b in zip(off[:-1], off[1:])]


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = np.max(np.abs(b)) if b.size else 0.0
    if scale > 0 and np.isfinite(scale):  # avoid overflow of the 2-norm (INEX reaches 1e177)
        a, b = a / scale, b / scale
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


@pytest.fixture(scope="session")
def gpu_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
