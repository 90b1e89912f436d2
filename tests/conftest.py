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
    """*_exact fixtures store only what differs from the base case."""
    g, s = load_golden(case)
    d = {k: g[k] for k in g.files}
    if case.endswith("_exact"):
        base, _ = load_golden(case[: -len("_exact")])
        for k in base.files:
            d.setdefault(k, base[k])
    return d, s


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


@pytest.fixture(scope="session")
def gpu_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
