"""End-to-end GPU setup parity: the device builds every
setup product itself; spectra, mode counts per subdomain, coarse dimension and
n_- must match the reference exactly, and the solve must match within the
north-star gates (iterations +-1, x within 1e-7).  Against the probe-fixed
oracle (exact pivoted factor, basis-invariant coarse solves) the applies also
match closely."""
import numpy as np
import pytest

from conftest import case_options, golden_with_base, one_level_of, rel
from paper_2106_10913_b200 import awg

pytestmark = pytest.mark.gpu

BASE = ["c1", "t2d", "t2d_ov2", "t3d", "t3d_blocks", "telas", "telas8", "tragged", "t1box"]


KINDS = {"NN": awg.OneLevelKind.NN, "AS": awg.OneLevelKind.AS, "AS_PLUS": awg.OneLevelKind.AS_PLUS}
COMPS = {"hybrid": awg.Composition.HYBRID, "additive": awg.Composition.ADDITIVE}
MODES = {"none": awg.AwgMode.NONE, "ad": awg.AwgMode.AD}


def setup_ctx(g, s, rrf="reference", options=None):
    n = len(g["b"])
    off, idx = g["part_offsets"], g["part_indices"]
    omega = [idx[a:b] for a, b in zip(off[:-1], off[1:])]
    a = awg.SparseSymMatrix(n, g["A_row_offsets"], g["A_col_indices"], g["A_values"])
    ctx = awg.ProblemContext(a, g["b"], awg.Partition(omega, n)).set_options(options)
    comp, mode = case_options(s)
    cfg = awg.PreconditionerConfig(rrf_semantics=rrf, one_level=KINDS[one_level_of(s)], composition=COMPS[comp],
                                   awg=MODES[mode], tau_flat=float(s.get("tau_flat", 10.0)))
    if s.get("fixed_k"):
        cfg.fixed_k = int(s["fixed_k"])
    else:
        cfg.tau_sharp = float(s["tau_sharp"])
    ctx.setup(cfg)
    return ctx


@pytest.mark.parametrize("case", BASE)
def test_setup_products(case):
    g, s = golden_with_base(case)
    ctx = setup_ctx(g, s)
    assert np.array_equal(ctx.get("n_nonpos"), g["n_nonpos"])
    assert np.array_equal(ctx.get("n_zero"), g["n_zero"])
    lam = ctx.get("lam")
    assert np.max(np.abs(lam - g["lam"])) <= 1e-10 * np.max(np.abs(g["lam"]))
    plam = ctx.get("pencil_lam")
    assert np.max(np.abs(plam - g["pencil_lam"])) <= 1e-8 * max(1.0, np.max(np.abs(g["pencil_lam"])))
    assert np.array_equal(ctx.get("ks"), g["ks"])
    q = ctx.query()
    assert q["n0"] == s["n0"] and q["n_minus"] == s["n_minus"]
    assert np.allclose(ctx.get("neg_weights"), g["neg_weights"], rtol=1e-9)
    # build_w's inner solves (continuously batched on the device) stop close to
    # where the reference's per-column pcg calls stop.  Under the reference's
    # pivoted-factor semantics H2 depends on the GenEO basis (bug 1 is not
    # basis invariant), and the device eigensolver's basis of a degenerate
    # cluster differs from Jacobi's, so counts move by up to 3 (measured); the
    # exact-semantics test below pins them to +-2.
    inner = ctx.get("w_inner_iterations")
    ref = np.asarray(g["w_inner_iterations"])
    assert inner.size == ref.size
    assert np.all(np.abs(inner - ref) <= np.maximum(3, 0.15 * ref)), (inner, ref)


@pytest.mark.parametrize("case", BASE + ["t2d_additive", "t3d_none", "t2d_as", "t2d_asplus", "telas_as"])
def test_solve_reference_semantics(case):
    g, s = golden_with_base(case)
    ctx = setup_ctx(g, s)
    x, rep = ctx.pcg(g["b"], s["rtol_solve"], 10000)
    assert rep.converged
    assert abs(rep.iterations - s["iterations"]) <= 1, (rep.iterations, s["iterations"])
    assert rel(x, g["pcg_x"]) <= 1e-7


@pytest.mark.parametrize("case", ["t2d_as", "t2d_asplus", "telas_as"])
def test_as_setup_products(case):
    """AS / AS+ coarse spaces: per-subdomain column counts (two pencils for AS,
    coarse.cpp:127-130) and the coarse dimension match the reference."""
    g, s = golden_with_base(case)
    ctx = setup_ctx(g, s)
    assert np.array_equal(ctx.get("ks"), g["ks"])
    q = ctx.query()
    assert q["n0"] == s["n0"] and q["n_minus"] == s["n_minus"]
    if "pencil_as1_lam" in g:
        assert np.max(np.abs(ctx.get("pencil_lam") - g["pencil_as1_lam"])) <= 1e-8 * max(
            1.0, np.max(np.abs(g["pencil_as1_lam"])))


@pytest.mark.parametrize("case", ["c1_exact", "t2d_exact"])
def test_exact_semantics_against_fixed_oracle(case):
    g, s = golden_with_base(case)
    ctx = setup_ctx(g, s, rrf="exact")
    for name, op in (("H1", awg.Op.H1), ("Q", awg.Op.Q), ("H2", awg.Op.H2), ("QW", awg.Op.QW)):
        for x, y in zip(g["x_apply"], g["y_" + name]):
            assert rel(ctx.apply(op, x), y) <= 1e-8, (case, name, rel(ctx.apply(op, x), y))
    xs, rep = ctx.pcg(g["b"], s["rtol_solve"], 10000)
    assert abs(rep.iterations - s["iterations"]) <= 1
    assert rel(xs, g["pcg_x"]) <= 1e-7
    # the batched W build keeps the per-column PCG semantics of build_w: every
    # inner solve stops at (nearly) the same iteration as the reference's
    inner = ctx.get("w_inner_iterations")
    assert inner.size == len(g["w_inner_iterations"])
    assert np.max(np.abs(inner - g["w_inner_iterations"])) <= 2, (inner, g["w_inner_iterations"])


def test_report_outputs(tmp_path):
    """run_with_context's report files (harness.cpp:151-224) from a GPU solve."""
    import json

    from paper_2106_10913_b200 import report

    g, s = golden_with_base("t2d")
    ctx = setup_ctx(g, s)
    x, rep = ctx.pcg(g["b"], s["rtol_solve"], 10000)
    r = report.write_outputs(str(tmp_path), "t2d run", ctx, ctx.cfg, rep, s["rtol_solve"], 10000)
    assert r["problem"]["coloring_A"] == s["coloring_A"]
    assert r["preconditioner"]["coarse_dim"] == s["n0"]
    assert r["solve"]["iterations"] == rep.iterations
    j = json.load(open(tmp_path / "t2d_run_report.json"))
    assert j["preconditioner"]["n_minus"] == s["n_minus"]
    lines = open(tmp_path / "rows.csv").read().splitlines()
    assert lines[0] == "label,kappa,it,lambda_min,lambda_max,v0,n_minus" and len(lines) == 2
    assert len(open(tmp_path / "t2d_run_residuals.csv").read().splitlines()) == rep.iterations + 1


def test_wide_coarse_blocks():
    """Subdomains with more than 64 coarse columns (k_bs_gemvT sweeps its
    columns in batches of 64): Q and A- on the device match the restatement
    evaluated on the factors the device built."""
    from oracle import awg_oracle as O

    g, s = golden_with_base("t3d")
    n = len(g["b"])
    omega = [g["part_indices"][a:b] for a, b in zip(g["part_offsets"][:-1], g["part_offsets"][1:])]
    a = awg.SparseSymMatrix(n, g["A_row_offsets"], g["A_col_indices"], g["A_values"])
    ctx = awg.ProblemContext(a, g["b"], awg.Partition(omega, n))
    cfg = awg.PreconditionerConfig()
    cfg.fixed_k = 70
    ctx.setup(cfg)
    ks = ctx.get("ks")
    assert ks.min() >= 70
    f = {k: ctx.get(k) for k in ("lam", "V", "n_nonpos", "n_zero", "ks", "Y", "k0_retained")}
    r0 = len(f["k0_retained"])
    f["k0_l11"] = ctx.get("k0_l11").reshape(r0, r0, order="F")  # column-major lower factor
    orc = O.AwgOracle(n, g["A_row_offsets"], g["A_col_indices"], g["A_values"], omega, f)
    rng = np.random.default_rng(11)
    for _ in range(3):
        x = rng.uniform(-1, 1, n)
        assert rel(ctx.apply(awg.Op.Q, x), orc.coarse_correct(x)) <= 1e-11
        assert rel(ctx.apply(awg.Op.AMINUS, x), orc.apply_Aminus(x)) <= 1e-11


@pytest.mark.parametrize("case", ["t3d", "telas8"])
def test_wbuild_grouped_dgemm_matches_cublas_path(case):
    """The W build's block one-level on the hand-written grouped FP64
    tensor-core GEMM (default) against the per-subdomain cuBLAS DGEMM path
    (option wbuild_cublas=1): same inner iteration counts (+-1) and the same W
    up to the inner solves' tolerance."""
    g, s = golden_with_base(case)
    ctx1 = setup_ctx(g, s)
    ctx2 = setup_ctx(g, s, options={"wbuild_cublas": 1})
    i1, i2 = ctx1.get("w_inner_iterations"), ctx2.get("w_inner_iterations")
    assert np.max(np.abs(i1.astype(int) - i2.astype(int))) <= 1
    w1, w2 = ctx1.get("W"), ctx2.get("W")
    assert rel(w1, w2) <= 1e-8


def test_not_spd_error_carries_the_reference_pivot():
    """cholesky (dense.cpp:226-249) throws NotSpdError(k) at the first
    non-positive pivot; the AS one-level factors R A R^T (preconditioner.cpp:
    20-30) hit it when A is indefinite.  t2d with the diagonal of dof 79 (owned
    by subdomain 0 alone, local index 46) set to -1: the unmodified reference
    (ref_driver --one-level AS) terminates with "matrix not spd: non-positive
    pivot at index 46"; the device's blocked factorisation must report the same
    pivot, through the same exception type."""
    g, s = golden_with_base("t2d_as")
    d = dict(g)
    vals = g["A_values"].copy()
    ro, ci = g["A_row_offsets"], g["A_col_indices"]
    i0 = 79
    for k in range(ro[i0], ro[i0 + 1]):
        if ci[k] == i0:
            vals[k] = -1.0
    d["A_values"] = vals
    # the restated unblocked factorisation on subdomain 0's block
    om0 = d["part_indices"][d["part_offsets"][0]:d["part_offsets"][1]]
    import scipy.sparse as sp
    a = sp.csr_matrix((vals, ci, ro), shape=(len(d["b"]),) * 2)[om0][:, om0].toarray()
    expect = None
    for k in range(a.shape[0]):
        if not a[k, k] > 0.0:
            expect = k
            break
        a[k + 1:, k] /= np.sqrt(a[k, k])
        a[k + 1:, k + 1:] -= np.outer(a[k + 1:, k], a[k + 1:, k])
    assert expect == 46
    with pytest.raises(awg.NotSpdError) as ei:
        setup_ctx(d, s)
    assert ei.value.pivot_index == 46
    assert "non-positive pivot at index 46" in str(ei.value)
