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


REF_DRIVER = __import__("os").path.join(__import__("os").path.dirname(__import__("os").path.dirname(
    __import__("os").path.abspath(__file__))), "oracle", "_ref", "ref_driver")
needs_ref = pytest.mark.skipif(not __import__("os").path.exists(REF_DRIVER), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("nx,ny,e,nu", [(9, 5, 1.0, 0.3), (17, 9, 1e7, 0.45), (33, 8, 2.5, 0.2)])
def test_elasticity_generator_matches_reference_assemble(tmp_path, nx, ny, e, nu):
    """problems.elasticity_problem with one material against the reference's
    own assemble() (fem.cpp:99-162, CoefficientField::constant, h = 1, load
    (0, -9.81); ref_driver --fem): same CSR pattern, values and rhs (summed in
    the same element order, sparse.cpp:19-47)."""
    import subprocess

    out = tmp_path / "fem"
    subprocess.run([REF_DRIVER, "--fem", str(nx), str(ny), repr(e), repr(nu), str(out)], check=True)
    ref = {k: np.load(out / f"{k}.npy") for k in ("row_offsets", "col_indices", "values", "b")}
    p = P.elasticity_problem("fem", nx, ny, 10 ** 6, [(e, nu)], (1, 1), 0)
    assert np.array_equal(p.row_offsets, ref["row_offsets"])
    assert np.array_equal(p.col_indices, ref["col_indices"])
    assert np.max(np.abs(p.values - ref["values"])) <= 1e-15 * np.max(np.abs(ref["values"]))
    assert np.max(np.abs(p.b - ref["b"])) <= 1e-15 * np.max(np.abs(ref["b"]))


def _bfs_owner(n, rp, ci, parts):
    """partition.cpp:42-77: BFS-grown parts of ~n/parts dofs (test-side
    restatement, used only to feed the same owners to both closures)."""
    from collections import deque

    part = -np.ones(n, dtype=np.int64)
    target = (n + parts - 1) // parts
    seed = 0
    for s in range(parts):
        while seed < n and part[seed] >= 0:
            seed += 1
        if seed >= n:
            break
        q = deque([seed])
        part[seed] = s
        grown, cap = 1, (n if s == parts - 1 else target)
        while q and grown < cap:
            i = q.popleft()
            for k in range(rp[i], rp[i + 1]):
                if grown >= cap:
                    break
                j = ci[k]
                if part[j] < 0:
                    part[j] = s
                    q.append(j)
                    grown += 1
    part[part < 0] = parts - 1
    return part


@needs_ref
@pytest.mark.parametrize("name,parts", [("t2d", 4), ("telas8", 3), ("t3d", 5)])
def test_overlap_closure_matches_reference(tmp_path, name, parts):
    """problems.overlap_closure (one ring) against the reference's own
    closure in auto_partition (partition.cpp:79-90; ref_driver --autopart) on
    the same BFS owners: identical index sets."""
    import subprocess

    p = P.make(name)
    prefix = str(tmp_path / name)
    p.write(prefix)
    out = tmp_path / "ap"
    subprocess.run([REF_DRIVER, "--autopart", prefix, str(parts), str(out)], check=True)
    off, idx = np.load(out / "part_offsets.npy"), np.load(out / "part_indices.npy")
    owner = _bfs_owner(p.n, p.row_offsets, p.col_indices, parts)
    ours = P.overlap_closure(p.n, p.row_offsets, p.col_indices, owner, parts, 1)
    for s in range(parts):
        assert np.array_equal(ours[s], idx[off[s]:off[s + 1]]), s
