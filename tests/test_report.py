"""Report quantities: the coloring bounds of the report
JSON against the unmodified reference (coloring_constant /
coloring_constant_aplus, partition.cpp:158-199, exported by ref_driver)."""
import pytest

from conftest import golden_with_base, omega_of
from paper_2106_10913_b200 import report


@pytest.mark.parametrize("case", ["c1", "t2d", "t2d_ov2", "t3d", "t3d_blocks", "telas"])
def test_colorings_match_reference(case):
    g, s = golden_with_base(case)
    omega = omega_of(g)
    n = len(g["b"])
    rp, ci = g["A_row_offsets"], g["A_col_indices"]
    assert report.coloring_constant(rp, ci, omega, n) == s["coloring_A"]
    has_neg = [(int(a) - int(b)) > 0 for a, b in zip(g["n_nonpos"], g["n_zero"])]
    assert report.coloring_constant_aplus(rp, ci, omega, n, has_neg) == s["coloring_Aplus"]
