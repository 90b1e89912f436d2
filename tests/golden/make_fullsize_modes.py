"""Full-size setup fixture: per-subdomain n_nonpos, n_zero and GenEO mode
counts of a BASELINE.json config at its full size, from the oracle
restatement (oracle/awg_oracle.py: build_Bs + eigsplit, weighted A+ and
R A+ R^T pencils, select_YL) — the reference's own setup takes 8-12 h at c2
(SURVEY.md §8c-4), the restatement's splitting and pencils minutes.  The
restatement is pinned to the reference on every golden case
(tests/test_oracle_golden.py); this extends the mode-count gate of
SURVEY.md §8c-2 to the full c2 size.  The margins (distance of the deciding
eigenvalues from eps_zero and from tau) are stored so a test can tell a
real mismatch from a tie.

    python tests/golden/make_fullsize_modes.py c2   ->  tests/golden/c2_modes.json
    python tests/golden/make_fullsize_modes.py c5 corner
        ->  tests/golden/c5_corner_modes.json: the 2x2x2 corner boxes only
            (their pencils need the eigensplits of the 3x3x3 boxes around
            them, not all 216 — a full c5 run is ~2.5 h of CPU)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import awg_oracle as O  # noqa: E402
from paper_2106_10913_b200 import problems  # noqa: E402


def main(name, subset=None):
    p = problems.make(name)
    a = O.csr(p.n, p.row_offsets, p.col_indices, p.values)
    omega = [np.asarray(o, dtype=np.int64) for o in p.omega]
    assert not O.check_minimal_overlap(a, omega)
    mult, _ = O.build_pou(omega, p.n)
    t0 = time.time()
    targets = list(range(len(omega)))
    need = set(targets)
    if subset == "corner":  # boxes (i, j, k) in {0,1}^3, lexicographic box order (x fastest)
        bx, by, _ = p.meta["boxes"]
        targets = [i + bx * j + bx * by * k for k in (0, 1) for j in (0, 1) for i in (0, 1)]
        marks = np.zeros(p.n, dtype=bool)
        for t in targets:
            marks[omega[t]] = True
        need = {s for s in range(len(omega)) if marks[omega[s]].any()}  # every subdomain overlapping a target
    mmu = O.entry_multiplicities(a, omega)
    ah = O.sp.csr_matrix((a.data / mmu, a.indices, a.indptr), shape=a.shape)
    bs = {s: ah[omega[s]][:, omega[s]].toarray() for s in sorted(need)}  # build_Bs on the needed subdomains
    empty = O.LocalSplit(np.zeros(0), np.zeros((0, 0)), 0, 0, 0.0)  # never overlaps a target
    splits, raw = [empty] * len(omega), {}
    for s in sorted(need):
        w, v = O.dense_sym_eig(bs[s])
        raw[s] = w.copy()
        splits[s] = O.eigsplit(w, v)
        print(f"eig {s}: {time.time() - t0:.0f} s", file=sys.stderr, flush=True)
    out = {"config": name, "n": p.n, "n_sub": len(omega), "tau_sharp": p.tau_sharp, "fixed_k": p.fixed_k,
           "subdomains": targets,
           "n_nonpos": [], "n_zero": [], "ks": [], "eps_margin": [], "tau_margin": [], "pencil_low": []}
    for s in targets:
        ls = splits[s]
        w = raw[s]
        eps = ls.eps_zero  # splitting.cpp:64-84; relative distance of the nearest raw eigenvalue to +-eps
        out["eps_margin"].append(float(np.min(np.minimum(np.abs(w - eps), np.abs(w + eps))) / eps))
        ma = O.weighted_asplus(bs[s], ls, mult[omega[s]].astype(np.float64))
        mb = O.local_Aplus_block(a, omega, splits, s)
        w, _ = O.generalized_sym_eig(ma, mb)
        k = O.select_count(w, p.tau_sharp, p.fixed_k, ls.n_nonpos)
        out["n_nonpos"].append(int(ls.n_nonpos))
        out["n_zero"].append(int(ls.n_zero))
        out["ks"].append(int(k))
        out["tau_margin"].append(float(np.min(np.abs(w - p.tau_sharp))) if p.tau_sharp else None)
        out["pencil_low"].append([float(v) for v in w[: k + 2]])
        print(f"pencil {s}: k = {k}, m = {ls.n_nonpos}, {time.time() - t0:.0f} s", file=sys.stderr, flush=True)
    if subset is None:
        out["n0"] = int(sum(out["ks"]))
        out["n_minus"] = int(sum(int(np.count_nonzero(ls.lam[: ls.n_nonpos] != 0.0)) for ls in splits))
    tag = f"{name}_{subset}" if subset else name
    with open(os.path.join(ROOT, "tests", "golden", f"{tag}_modes.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({k: out[k] for k in ("ks", "n_nonpos")}))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c2", sys.argv[2] if len(sys.argv) > 2 else None)
