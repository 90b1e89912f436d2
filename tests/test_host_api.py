"""The C++ host API (include/awg_b200/awg.hpp) over the C ABI: a C++ caller
compiles and links against libawg_b200.so here; on the GPU it runs the
reference's run_with_context pathway end to end."""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden_with_base, rel
from paper_2106_10913_b200 import awg, problems

SRC = os.path.join(ROOT, "tests", "cpp", "host_api_main.cpp")


def build_exe(tmp_path):
    exe = str(tmp_path / "host_api_main")
    libdir = os.path.dirname(awg.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
                    "-L" + libdir, "-lawg_b200", "-Wl,-rpath," + libdir], check=True)
    return exe


def test_cpp_host_api_builds(tmp_path):
    assert os.path.exists(build_exe(tmp_path))


@pytest.mark.gpu
def test_cpp_host_api_runs(tmp_path):
    exe = build_exe(tmp_path)
    g, s = golden_with_base("t2d")
    p = problems.make("t2d")
    assert np.array_equal(p.values, g["A_values"])
    prefix = str(tmp_path / "t2d")
    with open(prefix + ".bin", "wb") as f:
        np.asarray([p.n, p.nnz, p.n_sub], dtype=np.int32).tofile(f)
        np.asarray(p.row_offsets, dtype=np.int32).tofile(f)
        np.asarray(p.col_indices, dtype=np.int32).tofile(f)
        np.asarray(p.values, dtype=np.float64).tofile(f)
        np.asarray(p.b, dtype=np.float64).tofile(f)
        np.asarray(p.part_offsets(), dtype=np.int32).tofile(f)
        np.asarray(p.part_indices(), dtype=np.int32).tofile(f)
    out = subprocess.run([exe, prefix, repr(p.tau_sharp)], check=True, capture_output=True, text=True).stdout
    r = json.loads(out)
    assert r["converged"] == 1 and abs(r["iterations"] - s["iterations"]) <= 1
    assert r["n0"] == s["n0"] and r["n_minus"] == s["n_minus"]
    x = np.loadtxt(prefix + ".x")
    assert rel(x, g["pcg_x"]) <= 1e-7
