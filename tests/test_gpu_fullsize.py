"""Full-size checks at BASELINE.json configs[1] (c2: n = 65,536, 16
subdomains, the default bench workload).  The reference needs 8-12 h of CPU
time for this setup, so parity at this size goes through
size-independent properties of the operators instead of golden vectors:

* SpMV bit-identical to the reference's row loop (sparse.cpp:49-56: ascending
  columns, separate multiply and add), restated in numpy;
* H3 (AD over NN-hybrid) linear, symmetric and positive — the hybrid H2
  (I - Q A+) H1 (I - A+ Q) + Q (preconditioner.cpp:64-82) and W KW+ W^T
  (preconditioner.cpp:149-221) are symmetric positive (semi-)definite;
* the single-pass local solve equals the two-pass GEMV pair and the other
  task split (static per-CTA shares vs the atomic queue), and is independent
  of the cross-task copy prefetch (bit for bit);
* setup products against the oracle restatement at full size
  (tests/golden/c2_modes.json, tests/golden/make_fullsize_modes.py): n_nonpos,
  n_zero and GenEO mode counts per subdomain, n0, n_-, the low pencil spectra;
* PCG converges, its recursive residual agrees with the true residual, and
  repeated solves are bit-identical (fixed-order reductions, no atomics in
  any sum)."""
import json
import os

import numpy as np
import pytest

from conftest import rel
from fullsize_parity import FullSize, check_applies, check_coarse_solves, check_pcg, record
from paper_2106_10913_b200 import awg, problems

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2fs():
    fs = FullSize("c2")
    yield fs
    fs.close()


@pytest.fixture(scope="module")
def c2(c2fs):
    return c2fs.p, c2fs.ctx


def _ctx_with(fs, options):
    """A context on the same (exported) factors as fs with experiment options:
    awg_load_factors instead of another setup (the options only change how the
    operators run)."""
    ctx = awg.context_from_problem(fs.p, options=options)
    ctx.load_factors(awg.config_for(fs.p), fs.f)
    return ctx


def _spmv_reference_order(p, x):
    """y_i = (((0 + a_i0 x_c0) + a_i1 x_c1) + ...), as sparse.cpp:49-56."""
    rp = p.row_offsets.astype(np.int64)
    cnt = np.diff(rp)
    y = np.zeros(p.n)
    for k in range(int(cnt.max())):
        rows = np.nonzero(cnt > k)[0]
        e = rp[rows] + k
        y[rows] = y[rows] + p.values[e] * x[p.col_indices[e]]
    return y


def _check_modes(p, ctx, name):
    with open(os.path.join(os.path.dirname(__file__), "golden", f"{name}_modes.json")) as fh:
        ref = json.load(fh)
    subs = ref.get("subdomains", list(range(p.n_sub)))
    assert ctx.get("n_nonpos")[subs].tolist() == ref["n_nonpos"]
    assert ctx.get("n_zero")[subs].tolist() == ref["n_zero"]
    assert ctx.get("ks")[subs].tolist() == ref["ks"]
    if "n0" in ref:
        q = ctx.query()
        assert q["n0"] == ref["n0"] and q["n_minus"] == ref["n_minus"]
    plam = ctx.get("pencil_lam")
    off = np.concatenate([[0], np.cumsum([o.size for o in p.omega])])
    for s, low in zip(subs, ref["pencil_low"]):
        # 1e-8 of the subdomain's spectrum scale (the golden cases' bound,
        # test_gpu_setup); the pencil's zero cluster (size n_zero, values
        # ~1e-9..1e-7 at c2's 1e6 contrast) is rounding noise of a singular
        # pencil in both eigensolvers: it only has to stay far below tau
        scale = max(1.0, float(np.max(np.abs(plam[off[s]:off[s + 1]]))))
        got, low = plam[off[s]:off[s] + len(low)], np.asarray(low)
        zero = np.abs(low) < 1e-6
        assert np.all(np.abs(got[zero]) < 1e-6), s
        assert np.max(np.abs(got[~zero] - low[~zero])) <= 1e-8 * scale, s


def test_setup_mode_counts_full_size(c2):
    p, ctx = c2
    _check_modes(p, ctx, "c2")


def test_apply_parity_full_size(c2fs):
    """Every operator of the path on the device's own c2 factors within 1e-11
    of the restatement (preconditioner.cpp:32-82, 149-221; splitting.cpp:119-147;
    coarse.cpp:156-166)."""
    record("c2_applies", check_applies(c2fs))


def test_coarse_solves_full_size(c2fs):
    """K0 / KW solves (the reference's stale-upper factors: rw < n_minus at c2)."""
    record("c2_coarse_solves", check_coarse_solves(c2fs))


def test_pcg_parity_full_size(c2fs):
    """The device PCG against the restatement's pcg on the same factors:
    iterations +-1, x within 1e-7 (krylov.cpp:36-124)."""
    record("c2_pcg", check_pcg(c2fs))


def test_spmv_bit_identical_full_size(c2):
    p, ctx = c2
    x = problems.uniform(7, p.n, -1.0, 1.0)
    assert np.array_equal(ctx.apply(awg.Op.A, x), _spmv_reference_order(p, x))


def test_h3_linear_symmetric_positive(c2):
    p, ctx = c2
    x = problems.uniform(11, p.n, -1.0, 1.0)
    y = problems.uniform(12, p.n, -1.0, 1.0)
    hx, hy = ctx.apply(awg.Op.H3, x), ctx.apply(awg.Op.H3, y)
    hxy = ctx.apply(awg.Op.H3, 0.75 * x - 2.5 * y)
    assert rel(hxy, 0.75 * hx - 2.5 * hy) <= 1e-11
    a, b = float(y @ hx), float(x @ hy)
    assert abs(a - b) <= 1e-10 * np.linalg.norm(x) * np.linalg.norm(hy)
    assert float(x @ hx) > 0.0 and float(y @ hy) > 0.0
    for op in (awg.Op.H1, awg.Op.H2, awg.Op.Q, awg.Op.QW, awg.Op.APLUS):
        ox, oy = ctx.apply(op, x), ctx.apply(op, y)
        assert abs(float(y @ ox) - float(x @ oy)) <= 1e-10 * np.linalg.norm(x) * np.linalg.norm(oy), op


def test_local_solve_variants_full_size(c2fs):
    p = c2fs.p
    base = _ctx_with(c2fs, None)
    xs = [problems.uniform(21 + i, p.n, -1.0, 1.0) for i in range(2)]
    ref = [base.apply(awg.Op.H1, x) for x in xs]
    q = base.query()
    assert q["nn_single_pass"] == 1
    two = _ctx_with(c2fs, {"nn_two_pass": 1})
    nopf = _ctx_with(c2fs, {"fused_prefetch": 0})
    flip = _ctx_with(c2fs, {"fused_static": 0 if q["nn_static_split"] else 1})
    pdl = _ctx_with(c2fs, {"pdl_local": 0})
    try:
        # the early trigger into the local solve and its pre-wait copies change
        # scheduling only
        for x in xs:
            assert np.array_equal(pdl.apply(awg.Op.H1, x), base.apply(awg.Op.H1, x))
            assert np.array_equal(pdl.apply(awg.Op.H3, x), base.apply(awg.Op.H3, x))
        xa, ra = pdl.pcg(p.b, p.rtol, 10000)
        xb, rb = base.pcg(p.b, p.rtol, 10000)
        assert ra.iterations == rb.iterations and np.array_equal(xa, xb)
        for x, y in zip(xs, ref):
            assert rel(two.apply(awg.Op.H1, x), y) <= 1e-13
            assert np.array_equal(nopf.apply(awg.Op.H1, x), y)
            # the other task split: different column chunks, same sums regrouped
            assert rel(flip.apply(awg.Op.H1, x), y) <= 1e-13
        # the loaded factors reproduce the set-up context's operators
        for x in xs:
            assert rel(base.apply(awg.Op.H3, x), c2fs.ctx.apply(awg.Op.H3, x)) <= 1e-13
    finally:
        for cx in (base, two, nopf, flip, pdl):
            cx.close()


def test_pcg_full_size(c2fs):
    p, ctx = c2fs.p, c2fs.ctx
    x1, rep1 = ctx.pcg(p.b, p.rtol, 10000)
    x2, rep2 = ctx.pcg(p.b, p.rtol, 10000)
    assert rep1.converged and rep1.iterations == rep2.iterations
    assert np.array_equal(x1, x2), "fixed-order reductions: repeated solves are bit-identical"
    true = np.linalg.norm(p.b - _spmv_reference_order(p, x1)) / np.linalg.norm(p.b)
    # the host's batch sizing (convergence-rate estimate vs plain doubling) only
    # schedules graph launches: the device state decides, results identical
    base = _ctx_with(c2fs, None)
    fixed = _ctx_with(c2fs, {"pcg_adaptive": 0})
    try:
        x3, rep3 = fixed.pcg(p.b, p.rtol, 10000)
        x4, rep4 = base.pcg(p.b, p.rtol, 10000)
    finally:
        fixed.close()
        base.close()
    assert rep3.iterations == rep4.iterations and np.array_equal(x3, x4)
    assert abs(true - rep1.final_relative_residual) <= 1e-6 * true  # krylov.cpp:98: the true residual
    assert true <= p.rtol or abs(true - rep1.recurrence_residual_at_exit) <= 1e-8  # krylov.cpp:93-101


@pytest.mark.parametrize("mode", ["hyb", "inex", "inex_exact_lu"])
def test_h3_variants_full_size(c2fs, mode):
    """AWG HYB and INEX (preconditioner.cpp:199-221) and the projections Pi3 /
    Pi3^T (preconditioner.cpp:161-183) on the device's own c2 factors against
    the restatement, 1e-11.  INEX under the reference's lu_solve (bug 2,
    dense.cpp:404-409) overflows on c2's 262 x 262 core — the reference's own
    c2 run prints NaN for it (profiles/r02e/c2_reference_factors_*.json) — so
    there the bug-compatible device path must be non-finite exactly when the
    restatement is, and the comparison proper runs with the exact LU."""
    p = c2fs.p
    lu = "exact" if mode == "inex_exact_lu" else "reference"
    cfg = awg.config_for(p, lu_semantics=lu)
    cfg.awg = awg.AwgMode.HYB if mode == "hyb" else awg.AwgMode.INEX
    ctx = awg.context_from_problem(p)
    ctx.load_factors(cfg, c2fs.f)
    orc = c2fs.orc
    out = {}
    try:
        orc.lu_exact, orc._core = (lu == "exact"), None
        for seed in (1000, 1001):
            x = problems.uniform(seed, p.n, -1.0, 1.0)
            got = ctx.apply(awg.Op.H3, x)
            with np.errstate(all="ignore"):
                ref = orc.h3(x, "hyb" if mode == "hyb" else "inex")
            if not np.isfinite(ref).all():
                assert mode == "inex" and not np.isfinite(got).all(), "bug-compatible INEX: both sides overflow"
                out["H3inex_nonfinite_both"] = 1.0
                continue
            out["H3" + mode] = max(out.get("H3" + mode, 0.0), rel(got, ref))
            if mode == "hyb":
                out["PI3"] = max(out.get("PI3", 0.0), rel(ctx.apply(awg.Op.PI3, x), orc.apply_pi3(x)))
                out["PI3T"] = max(out.get("PI3T", 0.0), rel(ctx.apply(awg.Op.PI3T, x), orc.apply_pi3_transpose(x)))
    finally:
        orc.lu_exact, orc._core = False, None
        ctx.close()
    record("c2_h3_" + mode, out)
    assert out, mode
    assert all(np.isfinite(v) and v <= (1.0 if k.endswith("_both") else 1e-11) for k, v in out.items()), out
