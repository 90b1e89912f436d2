"""Golden vectors for the pivoted factor (TEST INFRASTRUCTURE).

Runs the UNMODIFIED reference's rank_revealing_sym_factor (dense.cpp:299-346,
oracle/_ref/ref_driver --rrf) and the probe-fixed one (oracle/_ref/ref_driver_fixed,
SURVEY.md §8c-3) on seeded symmetric matrices that exercise every branch of
the algorithm and stores G, retained and l11 of both in rrf_cases.npz:

  spd12_s*   random 12 x 12 SPD (SURVEY.md §0.4's probe shape: the reference's
             stale-upper swap loses rank there)
  spd64      a larger random SPD with a spread spectrum
  psd40r25   rank-deficient PSD (the drop rule piv <= 1e-10 * first)
  ties24     unit diagonal Gram matrix (every diagonal ties: first-maximum rule)
  ill30      graded SPD (pivots spanning 12 orders of magnitude)

    python tests/golden/make_rrf_golden.py
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(ROOT, "oracle", "_ref")


def cases():
    out = {}
    for seed in range(4):
        r = np.random.default_rng(100 + seed)
        b = r.standard_normal((12, 12))
        out[f"spd12_s{seed}"] = b @ b.T + 1e-3 * np.eye(12)
    r = np.random.default_rng(7)
    q, _ = np.linalg.qr(r.standard_normal((64, 64)))
    out["spd64"] = (q * np.logspace(-4, 2, 64)) @ q.T
    b = np.random.default_rng(8).standard_normal((40, 25))
    out["psd40r25"] = b @ b.T
    v = np.random.default_rng(9).standard_normal((24, 40))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    out["ties24"] = v @ v.T
    q, _ = np.linalg.qr(np.random.default_rng(10).standard_normal((30, 30)))
    out["ill30"] = (q * np.logspace(-12, 0, 30)) @ q.T
    return {k: 0.5 * (m + m.T) for k, m in out.items()}


def run(driver: str, g: np.ndarray, td: str):
    path = os.path.join(td, "g.bin")
    with open(path, "wb") as f:
        np.asarray([g.shape[0]], dtype=np.int32).tofile(f)
        np.asfortranarray(g).T.reshape(-1).tofile(f)  # column-major
    out = os.path.join(td, "out")
    subprocess.run([os.path.join(REF, driver), "--rrf", path, out], check=True)
    ret = np.load(os.path.join(out, "retained.npy"))
    l11 = np.load(os.path.join(out, "l11.npy"))
    return ret, l11


def main():
    blob = {}
    names = []
    with tempfile.TemporaryDirectory() as td:
        for name, g in cases().items():
            names.append(name)
            blob[f"{name}_G"] = g
            for tag, drv in (("ref", "ref_driver"), ("exact", "ref_driver_fixed")):
                ret, l11 = run(drv, g, td)
                blob[f"{name}_{tag}_retained"] = ret
                blob[f"{name}_{tag}_l11"] = l11
                print(f"{name:10s} {tag:5s} rank {len(ret)}/{g.shape[0]}")
    blob["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "rrf_cases.npz"), **blob)


if __name__ == "__main__":
    main()
