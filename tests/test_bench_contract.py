"""bench.py contract pieces that run without a GPU: the reference arm (the
compiled reference oracle on the host CPU) prints one valid JSON line."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "oracle", "_ref", "ref_driver")


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built")
def test_reference_arm_c1():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "applies/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] == 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_iteration_bytes_formula():
    import bench

    q = {"sum_ns2": 100, "sum_ns_ms": 10, "sum_ns": 10, "sum_ns_ks": 5, "r0": 2, "sum_ns_qs": 3, "n_minus": 1, "rw": 1}
    b = bench.iteration_bytes(q, n=10, nnz=30)
    b_spmv = 12 * 30 + 4 * 11 + 160
    expect = (3 * b_spmv + (8 * 2 * 90 + 8 * 3 * 10 + 80) + 2 * (16 * 5 + 8 * 4 + 160) + 2 * (8 * 3 + 160)
              + (16 * 10 + 8 + 160) + 8 * 16 * 10)
    assert b == expect
