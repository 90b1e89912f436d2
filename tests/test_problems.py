"""Workload generators (BASELINE.json configs and analogues)."""
import numpy as np
import pytest

from paper_2106_10913_b200 import problems as P
from oracle import awg_oracle as O


def test_splitmix64_reference_values():
    # SplitMix64 reference stream for seed 0 (Vigna's published generator).
    z = P.splitmix64(0, 3)
    assert [int(v) for v in z] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


@pytest.mark.parametrize("name,n,nnz,N,sizes", [
    ("c1", 1024, 4992, 4, (288, 288)),
    ("c2", 65536, 326656, 16, (4353, 4612)),
    ("c3", 262144, 1810432, 64, (4864, 5632)),
    ("c4", 130816, 2339368, 32, (4224, 4488)),
    ("c5", 884736, 6137856, 216, (4864, 5632)),
])
def test_config_sizes(name, n, nnz, N, sizes):
    """Sizes of SURVEY.md §8 table."""
    p = P.make(name)
    assert (p.n, p.nnz, p.n_sub) == (n, nnz, N)
    ns = [len(o) for o in p.omega]
    assert (min(ns), max(ns)) == sizes


@pytest.mark.parametrize("name", P.ANALOGUES + ["c1"])
def test_structure(name):
    p = P.make(name)
    a = O.csr(p.n, p.row_offsets, p.col_indices, p.values)
    assert abs(a - a.T).max() == 0.0  # bit-symmetric
    for i in range(p.n):
        c = p.col_indices[p.row_offsets[i]:p.row_offsets[i + 1]]
        assert np.all(np.diff(c) > 0)
    assert O.check_minimal_overlap(a, p.omega) == []
    for om in p.omega:
        assert np.all(np.diff(om) > 0)
    assert np.all(np.linalg.eigvalsh(a.toarray()) > 0)


def test_file_roundtrip(tmp_path):
    p = P.make("t2d")
    p.write(str(tmp_path / "t"))
    lines = open(tmp_path / "t.mtx").read().splitlines()
    assert lines[0] == "%%MatrixMarket matrix coordinate real symmetric"
    n, _, nl = map(int, lines[1].split())
    vals = {}
    for ln in lines[2:]:
        i, j, v = ln.split()
        vals[(int(i) - 1, int(j) - 1)] = float(v)
    d = p.dense()
    for (i, j), v in vals.items():
        assert d[i, j] == v and d[j, i] == v
    parts = [list(map(int, ln.split())) for ln in open(tmp_path / "t.part").read().splitlines()]
    assert [len(x) for x in parts] == [len(o) for o in p.omega]
