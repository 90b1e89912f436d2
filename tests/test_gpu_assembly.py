"""GPU-side problem assembly: the device builds the
benchmark systems and partitions bit-identically to the host generators
(problems.py, which restate the SURVEY §8d rules and, for elasticity, the
reference's assemble(), proj/src/fem.cpp:99-162 with TripletBuilder's
summation order, sparse.cpp:19-47), at every BASELINE.json size."""
import numpy as np
import pytest

from conftest import golden_with_base
from paper_2106_10913_b200 import awg, problems

pytestmark = pytest.mark.gpu

NAMES = ["c1", "t2d", "t2d_ov2", "t3d", "t3d_blocks", "telas", "telas8", "c2", "c3", "c4", "c5"]


@pytest.mark.parametrize("name", NAMES)
def test_device_assembly_matches_host(name):
    host = problems.make(name)
    ctx = awg.context_from_spec(problems.spec(name))
    try:
        assert ctx.a.n == host.n
        assert np.array_equal(ctx.a.row_offsets, host.row_offsets)
        assert np.array_equal(ctx.a.col_indices, host.col_indices)
        assert np.array_equal(ctx.a.values, host.values), "values must be bit-identical"
        assert ctx.partition.count() == host.n_sub
        for om_d, om_h in zip(ctx.partition.omega, host.omega):
            assert np.array_equal(om_d, om_h)
        assert np.array_equal(ctx.b, host.b)
    finally:
        ctx.close()


@pytest.mark.parametrize("case", ["telas8", "t2d"])
def test_device_assembly_matches_golden_and_solves(case):
    """The committed fixtures were generated from the host generator through
    the unmodified reference: the device-assembled system is the same system,
    and the GPU setup + solve on it gives the reference's iteration count."""
    g, s = golden_with_base(case)
    ctx = awg.context_from_spec(problems.spec(case))
    try:
        assert np.array_equal(ctx.a.values, g["A_values"])
        assert np.array_equal(ctx.b, g["b"])
        cfg = awg.PreconditionerConfig(tau_sharp=float(s["tau_sharp"]))
        ctx.setup(cfg)
        x, rep = ctx.pcg(ctx.b, s["rtol_solve"], 10000)
        assert rep.converged and abs(rep.iterations - s["iterations"]) <= 1
    finally:
        ctx.close()


def test_partition_owner_and_errors():
    host = problems.make("t3d")
    ctx = awg.context_from_spec(problems.spec("t3d"))
    try:
        # explicit owners: every dof its own box gives the same Omega^s as the boxes
        owner = np.zeros(host.n, dtype=np.int32)
        for s, om in enumerate(problems.overlap_closure(host.n, host.row_offsets, host.col_indices,
                                                        problems._box_owner((8, 8, 8), (2, 2, 2)), 8, 0)):
            owner[om] = s
        lib = ctx._lib
        rc = lib.awg_partition_owner(ctx._h, awg._ptr(owner, awg.ctypes.c_int), 8, 1)
        assert rc == awg.AWG_OK
        off = ctx.get("part_offsets")
        idx = ctx.get("part_indices")
        for s in range(8):
            assert np.array_equal(idx[off[s]:off[s + 1]], host.omega[s])
        bad = np.full(host.n, 9, dtype=np.int32)
        assert lib.awg_partition_owner(ctx._h, awg._ptr(bad, awg.ctypes.c_int), 8, 1) == awg.AWG_E_ARG
    finally:
        ctx.close()
    # boxes need a device-assembled matrix
    a = awg.SparseSymMatrix(host.n, host.row_offsets, host.col_indices, host.values)
    ext = awg.ProblemContext(a, host.b, awg.Partition(list(host.omega), host.n))
    try:
        bx = np.array([2, 2, 2], dtype=np.int32)
        assert ext._lib.awg_partition_boxes(ext._h, awg._ptr(bx, awg.ctypes.c_int), 1) == awg.AWG_E_STATE
    finally:
        ext.close()
    with pytest.raises(ValueError):
        awg.ProblemContext.assemble_fd((4,), np.ones(4), np.ones(4), (1,), 1)
