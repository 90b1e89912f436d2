"""The setup's hand-written batched symmetric eigensolver (csrc/eig.cu:
Householder tridiagonalisation with a TMA-streamed symmetric product,
bisection, twisted-factorisation vectors with inverse iteration on clusters,
WY back-transformation on the FP64 tensor cores) on seeded matrices, checked
against cuSOLVER Dsyevd on the same matrices (awg_bench_eig).  It replaces
the reference's cyclic Jacobi (dense_sym_eig, dense.cpp:117-209): eigenvalues
to rounding of ||A||, residuals ||A z - w z|| and orthogonality to ~1e-12."""
import pytest

from paper_2106_10913_b200 import awg

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,count,kind", [(2, 3, 0), (3, 2, 0), (65, 3, 0), (130, 2, 2), (300, 4, 0), (289, 2, 1), (1024, 2, 3),
                                          (1024, 3, 0), (1089, 2, 1), (2113, 2, 2)])
def test_eig_against_cusolver(n, count, kind):
    r = awg.bench_eig(n, count, kind, seed=7)
    assert r["eig_err"] <= 1e-13, r
    assert r["resid"] <= 1e-12, r
    assert r["orth"] <= 1e-11, r


@pytest.mark.parametrize("split", [0, 3, 8])
@pytest.mark.parametrize("n,count,kind", [(65, 3, 0), (300, 4, 0), (1089, 2, 1), (2113, 2, 2)])
def test_eig_both_panel_forms(n, count, kind, split):
    """One CTA per problem (k_latrd, eig_split = 0: what batches of >= 74
    problems take) and the split form with C CTAs per symmetric product
    (k_col_step + k_symv_part, the default for small batches) are the same
    algorithm; both meet the bounds."""
    r = awg.bench_eig(n, count, kind, seed=11, options={"eig_split": split})
    assert r["eig_err"] <= 1e-13, r
    assert r["resid"] <= 1e-12, r
    assert r["orth"] <= 1e-11, r
