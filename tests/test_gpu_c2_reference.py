"""BASELINE.json configs[1] (c2) end to end against runs of the reference
itself (tests/golden/c2_reference*.{npz,json}, made by
oracle/run_memo_reference.sh + tests/golden/make_c2_reference_golden.py: the
reference's own dense_sym_eig / generalized_sym_eig / pcg results memoised by
content hash — 23 h of one core —, then the stock ProblemContext +
run_with_context composition, harness.cpp:63-139):

* ``c2_reference``: the unmodified reference (shipped pivoted factor);
* ``c2_reference_exact``: the same objects with the probe-fixed pivoted
  factor (oracle/rrf_fixed.cpp).

The GPU path runs its own setup (Householder eigensolver instead of the
reference's cyclic Jacobi), so what can agree exactly are the integers
(n_nonpos, n_zero, GenEO mode counts, n0, r0, n_minus) and, to the accuracy of
the two eigensolvers, the basis-invariant operators H1, A- and A+.  H3 and the
solve go through K_W = W^T A W's pivoted factor.  With the exact factor that
is well-posed and the north-star gates apply (iterations +-1, x within 1e-7).
With the shipped factor (bug 1, dense.cpp:313-338) K_W loses 21 of its 262
columns at c2 and WHICH ones depends on rounding-level ties: the device's own
iteration count moved 95 -> 101 -> 128 across eigensolver revisions with every
operator still within 5e-15 of the restatement on the same factors
(test_gpu_fullsize.py), and the reference itself lands at 114.  There the
gates are the counts, the basis-invariant operators and convergence; the
iteration counts are recorded."""
import json
import os

import numpy as np
import pytest

from conftest import rel
from fullsize_parity import record
from paper_2106_10913_b200 import awg, problems

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
VARIANTS = {k: v for k, v in {"c2_reference": "reference", "c2_reference_exact": "exact"}.items()
            if os.path.exists(os.path.join(GOLD, k + ".json"))}  # (a golden is a 20+ h offline reference run)


def _load(name):
    with open(os.path.join(GOLD, name + ".json")) as fh:
        meta = json.load(fh)
    return meta, np.load(os.path.join(GOLD, name + ".npz"))


@pytest.fixture(scope="module", params=list(VARIANTS))
def run(request):
    name = request.param
    meta, g = _load(name)
    p = problems.make("c2")
    ctx = awg.context_from_problem(p)
    ctx.setup(awg.config_for(p, rrf_semantics=VARIANTS[name]))
    yield name, p, ctx, meta, g
    ctx.close()


def test_setup_counts_identical(run):
    """splitting.cpp:64-105 (eigsplit), coarse.cpp:113-154 (selection),
    dense.cpp:299-346 (retained ranks)."""
    name, p, ctx, meta, g = run
    assert meta["n"] == p.n and meta["n_sub"] == p.n_sub
    assert np.array_equal(ctx.get("n_nonpos"), g["n_nonpos"])
    assert np.array_equal(ctx.get("n_zero"), g["n_zero"])
    assert np.array_equal(ctx.get("ks"), g["ks"])
    q = ctx.query()
    got = {k: q[k] for k in ("n0", "r0", "n_minus", "rw")}
    record(name + "_counts", {"device": got, "reference": {k: meta[k] for k in got}})
    assert got["n0"] == meta["n0"] and got["n_minus"] == meta["n_minus"] and got["r0"] == meta["r0"]
    if VARIANTS[name] == "exact":
        assert got["rw"] == meta["rw"]
    else:  # shipped factor: which near-tie pivots drop is rounding-dependent
        assert abs(got["rw"] - meta["rw"]) <= 8, (got, meta["rw"])


def test_basis_invariant_operators(run):
    """The reference's applies on its own factors vs the device's on its own:
    H1 = sum R^T D P^s D R, A- and A+ do not depend on the eigenvector basis,
    so they agree to the accuracy of the two eigensolvers.  H1 is a
    pseudo-inverse (error ~ 1 / lambda_min+) and both eigensolvers are normwise
    (the reference's Jacobi: vector residuals 2e-9, eigenvalues second-order
    accurate; Householder + bisection: smaller residuals, eigenvalues 2e-8 ..
    6e-8 relative on the smallest positive modes): LAPACK's P^s x differs from
    the reference's by 9.6e-9 (profiles/r02e/h1_accuracy_c2.txt).  Measured
    here: H1 5.8e-9, A- 9.6e-12, A+ 4.9e-14."""
    name, p, ctx, meta, g = run
    out = {}
    for op, key in ((awg.Op.H1, "y_H1"), (awg.Op.AMINUS, "y_Aminus"), (awg.Op.APLUS, "y_Aplus"), (awg.Op.H3, "y_H3ad")):
        for x, y in zip(g["x_apply"], g[key]):
            out[key] = max(out.get(key, 0.0), rel(ctx.apply(op, x), y))
    record(name + "_operators", out)
    assert out["y_Aplus"] <= 1e-11 and out["y_Aminus"] <= 1e-10 and out["y_H1"] <= 2e-8, out
    if VARIANTS[name] == "exact":
        assert out["y_H3ad"] <= 1e-7, out  # W known to w_rtol = 1e-10 on each side


def test_pcg_against_reference(run):
    """krylov.cpp:36-124 through harness.cpp:131-139."""
    name, p, ctx, meta, g = run
    x, rep = ctx.pcg(p.b, p.rtol, 10 * p.n)
    info = {"iterations": rep.iterations, "reference_iterations": meta["iterations"], "x_rel": rel(x, g["pcg_x"]),
            "kappa": rep.kappa_estimate, "reference_kappa": meta["kappa"],
            "final_relres": rep.final_relative_residual, "reference_final_relres": meta["final_relative_residual"],
            "reference_t_h3_apply_s": meta["t_h3_apply"], "reference_t_solve_s": meta["t_solve"],
            "reference_serial_setup_s": sum(v for k, v in meta["serial_setup_s"].items() if k != "calls")}
    record(name + "_pcg", info)
    assert rep.converged and meta["converged"]
    assert rep.final_relative_residual <= p.rtol or abs(rep.final_relative_residual -
                                                         rep.recurrence_residual_at_exit) <= 1e-8
    if VARIANTS[name] == "exact":
        assert abs(rep.iterations - meta["iterations"]) <= 1, info
        assert info["x_rel"] <= 1e-7, info
        assert abs(rep.kappa_estimate - meta["kappa"]) <= 1e-3 * meta["kappa"], info
    else:
        # ill-posed under bug 1 (see the module docstring): both solves reach rtol;
        # the iteration counts stay within the spread the device itself has shown
        assert abs(rep.iterations - meta["iterations"]) <= 0.25 * meta["iterations"], info
        assert info["x_rel"] <= 1e-6, info


def test_w_inner_iterations(run):
    """build_w's inner PCG(A+, H2) per W column (preconditioner.cpp:97-113).
    The right-hand side of column (s, k) is R^s^T v_k: c2's negative spectra
    are (nearly) degenerate by the problem's symmetry, so v_k — and with it the
    single column's iteration count — depends on the eigensolver's basis of
    that eigenspace (measured: up to 9 of ~24 iterations on single columns,
    198 of 262 columns differ); the work as a whole does not: totals within
    4% (6,238 vs 6,441 shipped, 5,325 vs 5,563 exact).  Gate: totals within
    10%, every column within a factor 2."""
    name, p, ctx, meta, g = run
    inner = ctx.get("w_inner_iterations")
    ref = np.asarray(g["w_inner_iterations"])
    assert inner.size == ref.size
    d = np.abs(inner - ref)
    record(name + "_w_inner", {"device_total": int(inner.sum()), "reference_total": int(ref.sum()),
                               "max_abs_diff": int(d.max()), "columns_differing": int((d > 0).sum())})
    assert abs(int(inner.sum()) - int(ref.sum())) <= 0.10 * ref.sum()
    assert np.all(inner <= 2 * ref) and np.all(ref <= 2 * inner), (inner, ref)


def test_device_eigenpair_residuals(run):
    """The B^s eigenpairs behind H1 (subdomain 5, the 20 smallest positive
    modes): residuals ||B v - lambda v|| and eigenvalues against their Rayleigh
    quotients, next to the same figures of the reference's own Jacobi
    eigenpairs and of LAPACK on the same matrix (profiles/r02e/h1_accuracy_c2.txt:
    reference residuals 2.0-2.3e-9 with eigenvalues equal to their Rayleigh
    quotients to 4e-14; LAPACK residuals 4e-10, eigenvalues 2e-8 relative).
    Device (measured): residuals 1e-13 .. 6.6e-9, eigenvalues within 6.2e-8
    relative (5e-16 ||B^s||).  Both sides are at eps ||B^s|| ~ 4e-10 .. 7e-9 in the
    residual; the H1 gap of 5.8e-9 is their combination."""
    import scipy.sparse as sp

    from oracle import awg_oracle as O

    name, p, ctx, meta, g = run
    if VARIANTS[name] != "reference":
        return  # the eigenpairs do not depend on the pivoted factor: checked once
    s = 5
    sizes = np.array([len(o) for o in p.omega], dtype=np.int64)
    ns, poff, voff = int(sizes[s]), int(sizes[:s].sum()), int((sizes[:s] ** 2).sum())
    V, lam = ctx.get("V"), ctx.get("lam")
    Vs = V[voff:voff + ns * ns].reshape(ns, ns, order="F")
    ls, m = lam[poff:poff + ns], int(g["n_nonpos"][s])
    a = O.csr(p.n, p.row_offsets, p.col_indices, p.values)
    ah = sp.csr_matrix((a.data / O.entry_multiplicities(a, p.omega), a.indices, a.indptr), shape=a.shape)
    om = p.omega[s]
    B = ah[om][:, om].tocsr()
    Z = Vs[:, m:m + 20]
    res = np.linalg.norm(B @ Z - Z * ls[m:m + 20], axis=0)
    rq = np.einsum("ij,ij->j", Z, B @ Z)
    bnorm = float(abs(B).sum(axis=1).max())
    info = {"residual_smallest_positive": float(res[0]), "residual_max_of_20": float(res.max()),
            "eigenvalue_vs_rayleigh_quotient_rel_max": float(np.max(np.abs(rq - ls[m:m + 20]) / ls[m:m + 20])),
            "orthogonality_of_20": float(np.abs(Z.T @ Z - np.eye(20)).max()), "norm_B": bnorm,
            "reference_residual_max_of_20": 2.29e-9, "lapack_residual_max_of_20": 1.34e-9}
    record(name + "_eigenpairs", info)
    assert res.max() <= 1e-14 * bnorm, info  # the eigensolver's residual bound (test_gpu_eig: 1.1e-14 ||A||)
    assert info["orthogonality_of_20"] <= 1e-11, info
