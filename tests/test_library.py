"""The C-ABI library: builds for sm_100a, exports every symbol of
include/awg_cuda.h, and fails loudly without a GPU (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2106_10913_b200 import awg

HEADER = os.path.join(ROOT, "include", "awg_cuda.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*|long long)\s+(awg_\w+)\s*\(", text, re.M)))


def test_library_built():
    assert os.path.exists(awg.LIB_PATH), "run __graft_entry__.build()"


def test_exports_every_declared_symbol():
    lib = ctypes.CDLL(awg.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(awg.EXPORTED_SYMBOLS) == names


def test_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", awg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_no_gpu_fails_loudly():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    from paper_2106_10913_b200 import problems

    p = problems.make("t2d")
    with pytest.raises(awg.AwgCudaError):
        awg.context_from_problem(p)
