"""BASELINE.json configs[2] at full size (64^3, 64 subdomains, fixed k = 10,
n = 262,144): the device setup's per-subdomain counts against the
restatement's full-size fixture, then every operator and the PCG on the
device's own factors against the restatement (fullsize_parity.py)."""
import pytest

from fullsize_parity import FullSize, check_applies, check_coarse_solves, check_pcg, record
from test_gpu_fullsize import _check_modes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3():
    fs = FullSize("c3")
    yield fs
    fs.close()


def test_setup_mode_counts_c3(c3):
    """n_nonpos / n_zero and the fixed-k rule k_s = max(10, n_nonpos) extended
    over clusters, per subdomain, against tests/golden/c3_modes.json."""
    _check_modes(c3.p, c3.ctx, "c3")


def test_apply_parity_c3(c3):
    record("c3_applies", check_applies(c3))


def test_coarse_solves_c3(c3):
    """r0 = 2,105: the explicit K+ against forward + back substitution."""
    record("c3_coarse_solves", check_coarse_solves(c3))


def test_pcg_parity_c3(c3):
    record("c3_pcg", check_pcg(c3))
