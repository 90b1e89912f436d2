"""BASELINE.json configs[4] — the north-star config (96^3, 216 subdomains,
fixed k = 8, n = 884,736) — at full size, un-gated.  The reference's shipped
pivoted factor makes the c5 solve ill-posed under rounding (
685 vs 679 iterations across two builds of the same path), so the end-to-end
gates run the exact (probe-fixed) semantics, where the
problem is well-posed:
* the corner subdomains' counts against the restatement's fixture
  (tests/golden/c5_corner_modes.json, the 2x2x2 corner boxes whose pencils
  need only the 27 surrounding eigensplits);
* every operator of the path on the device's own factors within 1e-11 of the
  restatement (V^s 50 GB and W 21 GB exported to the host);
* the K0 / KW solves (rank ~2,900) against forward + back substitution;
* the device PCG against the restatement's pcg on the same factors."""
import pytest

from fullsize_parity import FullSize, check_applies, check_coarse_solves, check_pcg, record
from test_gpu_fullsize import _check_modes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c5():
    fs = FullSize("c5", rrf="exact")
    record("c5_setup", {"setup_s": fs.setup_s, **{k: fs.ctx.query()[k] for k in ("n0", "r0", "n_minus", "rw")}})
    yield fs
    fs.close()


def test_setup_mode_counts_c5_corner(c5):
    _check_modes(c5.p, c5.ctx, "c5_corner")


def test_apply_parity_c5(c5):
    record("c5_applies", check_applies(c5, seeds=(1000,)))


def test_coarse_solves_c5(c5):
    record("c5_coarse_solves", check_coarse_solves(c5))


def test_pcg_parity_c5(c5):
    record("c5_pcg", check_pcg(c5))
