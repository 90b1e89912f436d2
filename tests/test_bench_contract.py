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


@pytest.mark.gpu
def test_bench_line_contract_c1():
    """One real bench.py run on the GPU (c1: seconds) carries every key the
    driver reads: metric / value / unit, the workload name, ms_per_step,
    roofline (bound, achieved, peak, frac, traffic), cpu_baseline (the
    reference on the host cores), e2e with its copy sizes, gpu_launches,
    clocks; the solves converged."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--steps", "3",
                          "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert "invalid" not in line
    assert line["unit"] == "applies/s" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3 and line["ms_per_step"] > 0
    assert line["config"]["workload"] == "c1" and line["dtype"] == "f64" and line["vs_baseline"] is None
    r = line["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) <= 1e-9 * max(1.0, r["frac"])
    assert "traffic" in r
    e = line["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 8 * line["config"]["n"] == e["d2h_bytes_per_step"]
    assert line["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"])
    assert line["solve"]["converged_all"] is True
    if os.path.exists(REF):
        assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["value"] > 0
