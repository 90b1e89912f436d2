"""Regenerate the committed golden fixtures (TEST INFRASTRUCTURE).

Each fixture is the output of the UNMODIFIED reference (oracle/_ref/ref_driver,
built from /root/reference/proj/src by oracle/Makefile) on a problem from
paper_2106_10913_b200/problems.py written in the reference's external formats:
the problem itself (CSR, b, partition), every exported setup product (B^s
spectra and eigenvectors, mode counts, GenEO vectors, K0, W, KW, ...), applies
of every operator on seeded vectors, and the PCG result.  ``*_exact`` cases run
the probe-fixed oracle (oracle/_ref/ref_driver_fixed).

    python tests/golden/make_golden.py [case ...]
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2106_10913_b200 import problems  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(ROOT, "oracle", "_ref")

# case -> (problem, driver binary, extra args, export dense pencil matrices, base case)
# Variants store only what differs from their base case (same problem, same
# B^s eigenpairs and pencils).
CASES = {
    "c1": ("c1", "ref_driver", [], False, None),
    "c1_exact": ("c1", "ref_driver_fixed", [], False, "c1"),
    "t2d": ("t2d", "ref_driver", [], False, None),
    "t2d_exact": ("t2d", "ref_driver_fixed", [], False, "t2d"),
    "t2d_additive": ("t2d", "ref_driver", ["--comp", "additive"], False, "t2d"),
    "t2d_ov2": ("t2d_ov2", "ref_driver", [], False, None),
    "t3d": ("t3d", "ref_driver", [], False, None),
    "t3d_none": ("t3d", "ref_driver", ["--awg", "none"], False, "t3d"),
    "t3d_blocks": ("t3d_blocks", "ref_driver", [], False, None),
    # edge cases: ragged boxes; a single subdomain (no negative modes: AWG = H2)
    "tragged": ("tragged", "ref_driver", [], False, None),
    "t1box": ("t1box", "ref_driver", [], False, None),
    "telas": ("telas", "ref_driver", [], True, None),
    "telas8": ("telas8", "ref_driver", [], False, None),
    # one-level AS / AS+ (Cholesky factor form, preconditioner.cpp:20-30) with their
    # coarse spaces (coarse.cpp:122-130): Y comes from other pencils, so it is kept
    "t2d_as": ("t2d", "ref_driver", ["--one-level", "AS", "--tau-flat", "10"], False, "t2d"),
    "t2d_asplus": ("t2d", "ref_driver", ["--one-level", "AS_PLUS", "--tau-flat", "10"], False, "t2d"),
    "telas_as": ("telas", "ref_driver", ["--one-level", "AS", "--tau-flat", "10"], False, "telas"),
}


def run_case(name: str) -> str:
    prob_name, driver, extra, dense, base = CASES[name]
    p = problems.make(prob_name)
    with tempfile.TemporaryDirectory() as td:
        prefix = os.path.join(td, prob_name)
        p.write(prefix)
        out = os.path.join(td, "out")
        args = [os.path.join(REF, driver), prefix, out, "--n-apply", "3"]
        args += ["--fixed-k", str(p.fixed_k)] if p.fixed_k else ["--tau", repr(p.tau_sharp)]
        args += ["--rtol", repr(p.rtol)]
        if dense:
            args += ["--export-dense", "1"]
        args += extra
        subprocess.run(args, check=True)
        data = {}
        for f in sorted(os.listdir(out)):
            if f.endswith(".npy"):
                data[f[:-4]] = np.load(os.path.join(out, f))
        with open(os.path.join(out, "summary.json")) as fh:
            summary = json.load(fh)
    data.pop("Z", None)  # dense Z is derivable from Y; keep fixtures small
    data.pop("v_minus", None)  # derivable from V and n_nonpos
    if base:
        # B^s eigenpairs and pencil vectors are those of the base case; the
        # coarse factors, W (inner H2 solves) and everything downstream are kept.
        for k in ["V", "lam", "pencil_lam"] + ([] if "--one-level" in extra else ["Y"]):
            data.pop(k, None)
    data["A_row_offsets"] = p.row_offsets
    data["A_col_indices"] = p.col_indices
    data["A_values"] = p.values
    data["b"] = p.b
    data["part_offsets"] = p.part_offsets()
    data["part_indices"] = p.part_indices()
    summary.update({"case": name, "problem": prob_name, "driver": driver, "base": base, "args": extra,
                    "tau_sharp": p.tau_sharp, "fixed_k": p.fixed_k, "rtol_solve": p.rtol})
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **data)
    with open(os.path.join(HERE, name + ".json"), "w") as fh:
        json.dump(summary, fh, indent=1, sort_keys=True)
    return path


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        path = run_case(nm)
        print(nm, os.path.getsize(path) // 1024, "KiB")
