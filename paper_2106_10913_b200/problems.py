"""Synthetic workloads for the AWG-PCG hot path (BASELINE.json configs c1..c5).

The reference ships no finite-difference generator and no box partitioner with
algebraic overlap; it consumes external systems through
``read_matrix_market`` / ``read_vector`` / ``read_partition``
(proj/src/sparse.cpp:89-138, proj/src/partition.cpp:212-233).  These
generators therefore *are* the workload.  They produce:

* a symmetric CSR matrix with both triangles stored and strictly increasing
  column indices per row (proj/include/awg/sparse.hpp:12-21), bit-symmetric
  (each coupling value is computed once and stored in both triangles);
* a right-hand side;
* overlapping subdomains: disjoint boxes grown by ``overlap`` rings of
  matrix-graph closure, the closure rule of proj/src/partition.cpp:79-90.

Conventions:
* RNG: SplitMix64(seed); u = (next() >> 11) * 2^-53; U[a,b] = a + (b-a) u;
  N(0,1) by Box-Muller on consecutive (u1, u2) pairs.
* Lexicographic ordering, x fastest.  Homogeneous Dirichlet; cell-centred
  coefficients, harmonic-mean face coefficients, a boundary face uses its cell
  coefficient.
* b = U[-1,1] over the dofs in order, seed 0 (elasticity: the body force).

Bitwise reproducibility holds for the same numpy build; parity fixtures under
tests/golden store A, b and the partition explicitly, so tests never depend
on transcendental-function rounding of the host.
"""
from __future__ import annotations

import dataclasses
import os
from typing import List, Optional

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int) -> np.ndarray:
    """First ``count`` outputs of SplitMix64 seeded with ``seed`` (uint64)."""
    with np.errstate(over="ignore"):
        k = np.arange(1, count + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + k * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, count: int) -> np.ndarray:
    return (splitmix64(seed, count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform(seed: int, count: int, a: float, b: float) -> np.ndarray:
    return a + (b - a) * uniform01(seed, count)


def normal(seed: int, count: int) -> np.ndarray:
    pairs = (count + 1) // 2
    u = uniform01(seed, 2 * pairs)
    u1, u2 = u[0::2], u[1::2]
    r = np.sqrt(-2.0 * np.log1p(-u1))  # 1-u1 in (0,1]: log finite
    z = np.empty(2 * pairs)
    z[0::2] = r * np.cos(2.0 * np.pi * u2)
    z[1::2] = r * np.sin(2.0 * np.pi * u2)
    return z[:count]


@dataclasses.dataclass
class Problem:
    """A linear system plus its overlapping partition (the reference's
    ProblemContext inputs, proj/include/awg/harness.hpp:73-98)."""

    name: str
    n: int
    row_offsets: np.ndarray  # int32 (n+1)
    col_indices: np.ndarray  # int32 (nnz)
    values: np.ndarray  # float64 (nnz)
    b: np.ndarray  # float64 (n)
    omega: List[np.ndarray]  # sorted int32 index sets
    tau_sharp: Optional[float] = 0.1  # NN threshold (None when fixed_k is used)
    fixed_k: Optional[int] = None
    rtol: float = 1e-8
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.col_indices.size)

    @property
    def n_sub(self) -> int:
        return len(self.omega)

    def part_offsets(self) -> np.ndarray:
        off = np.zeros(self.n_sub + 1, dtype=np.int64)
        off[1:] = np.cumsum([o.size for o in self.omega])
        return off

    def part_indices(self) -> np.ndarray:
        return np.concatenate(self.omega).astype(np.int32)

    def dense(self) -> np.ndarray:
        d = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.row_offsets))
        d[rows, self.col_indices] = self.values
        return d

    # -- file exchange in the reference's external formats ------------------
    def write(self, prefix: str) -> None:
        """prefix.mtx / .rhs / .part as read by sparse.cpp:89-138 and
        partition.cpp:212-233 (values printed %.17g: bit-exact round trip)."""
        d = os.path.dirname(prefix)
        if d:
            os.makedirs(d, exist_ok=True)
        rows = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_offsets))
        lower = self.col_indices <= rows
        r, c, v = rows[lower] + 1, self.col_indices[lower].astype(np.int64) + 1, self.values[lower]
        with open(prefix + ".mtx", "w") as f:
            f.write("%%MatrixMarket matrix coordinate real symmetric\n")
            f.write(f"{self.n} {self.n} {int(lower.sum())}\n")
            f.write("".join(f"{a} {b_} {repr(float(x))}\n" for a, b_, x in zip(r.tolist(), c.tolist(), v.tolist())))
        with open(prefix + ".rhs", "w") as f:
            f.write(f"{self.n}\n")
            f.write("".join(f"{repr(float(x))}\n" for x in self.b.tolist()))
        with open(prefix + ".part", "w") as f:
            for om in self.omega:
                f.write(" ".join(map(str, om.tolist())) + "\n")


# ---------------------------------------------------------------------------
# Finite-difference diffusion on a cell grid


def _fd_matrix(shape, coeff: np.ndarray):
    """5-point (2D) / 7-point (3D) cell-centred diffusion stencil.

    shape = (nx, ny) or (nx, ny, nz); coeff flattened lexicographically, x
    fastest.  A_ij = -c_face for face neighbours, A_ii = sum of the cell's face
    coefficients (boundary faces use the cell coefficient)."""
    dims = len(shape)
    n = int(np.prod(shape))
    c = coeff.reshape(tuple(reversed(shape)))  # (nz, ny, nx) / (ny, nx)
    strides = [1]
    for s in shape[:-1]:
        strides.append(strides[-1] * s)
    # Face coefficients per axis: faces between cell and its +neighbour.
    face = []
    for ax in range(dims):
        npax = dims - 1 - ax  # numpy axis of grid axis ax
        lo = [slice(None)] * dims
        hi = [slice(None)] * dims
        lo[npax] = slice(0, -1)
        hi[npax] = slice(1, None)
        c1, c2 = c[tuple(lo)], c[tuple(hi)]
        face.append((2.0 * c1 * c2) / (c1 + c2))
    diag = np.zeros_like(c)
    offd = {}  # (ax, sign) -> coefficient array over all cells (nan = absent)
    for ax in range(dims):
        npax = dims - 1 - ax
        f = face[ax]
        minus = np.full_like(c, np.nan)
        plus = np.full_like(c, np.nan)
        sl_hi = [slice(None)] * dims
        sl_hi[npax] = slice(1, None)
        sl_lo = [slice(None)] * dims
        sl_lo[npax] = slice(0, -1)
        minus[tuple(sl_hi)] = f
        plus[tuple(sl_lo)] = f
        offd[(ax, -1)] = minus
        offd[(ax, +1)] = plus
    # Diagonal: faces summed in the order -x,+x,-y,+y(,-z,+z).
    for ax in range(dims):
        for sgn in (-1, 1):
            f = offd[(ax, sgn)]
            diag = diag + np.where(np.isnan(f), c, f)
    idx = np.arange(n, dtype=np.int64)
    slots_cols, slots_vals = [], []
    # Ascending column order: -z, -y, -x, self, +x, +y, +z.
    order = [(ax, -1) for ax in reversed(range(dims))] + [None] + [(ax, +1) for ax in range(dims)]
    for key in order:
        if key is None:
            slots_cols.append(idx)
            slots_vals.append(diag.reshape(-1))
        else:
            ax, sgn = key
            v = offd[key].reshape(-1)
            slots_cols.append(idx + sgn * strides[ax])
            slots_vals.append(-v)
    cols = np.stack(slots_cols, axis=1)
    vals = np.stack(slots_vals, axis=1)
    valid = ~np.isnan(vals)
    counts = valid.sum(axis=1)
    row_offsets = np.zeros(n + 1, dtype=np.int64)
    row_offsets[1:] = np.cumsum(counts)
    return (row_offsets.astype(np.int32), cols[valid].astype(np.int32), vals[valid].astype(np.float64))


def _pattern(n, row_offsets, col_indices):
    import scipy.sparse as sp

    return sp.csr_matrix(
        (np.ones(col_indices.size, dtype=np.float32), col_indices, row_offsets.astype(np.int64)), shape=(n, n)
    )


def overlap_closure(n, row_offsets, col_indices, owner: np.ndarray, n_sub: int, rings: int) -> List[np.ndarray]:
    """Disjoint parts grown by ``rings`` rings of matrix-graph closure (every
    stored coupling of a member joins; proj/src/partition.cpp:79-90)."""
    import scipy.sparse as sp

    p = _pattern(n, row_offsets, col_indices)
    ind = sp.csr_matrix(
        (np.ones(n, dtype=np.float32), (np.arange(n), owner.astype(np.int64))), shape=(n, n_sub)
    )
    m = ind
    for _ in range(rings):
        m = ((p @ m) + m)
        m.data[:] = 1.0
    m = m.tocsc()
    m.sort_indices()
    out = []
    for s in range(n_sub):
        out.append(np.asarray(m.indices[m.indptr[s]:m.indptr[s + 1]], dtype=np.int32))
    return out


def _box_owner(shape, boxes):
    """Owner subdomain per cell of a regular box decomposition; subdomains
    numbered lexicographically, x fastest."""
    grids = np.meshgrid(*[np.arange(s) for s in reversed(shape)], indexing="ij")
    owner = np.zeros(grids[0].shape, dtype=np.int64)
    mult = 1
    for ax in range(len(shape)):
        coord = grids[len(shape) - 1 - ax]
        w = shape[ax] // boxes[ax]
        owner += np.minimum(coord // w, boxes[ax] - 1) * mult  # the last box takes the remainder
        mult *= boxes[ax]
    return owner.reshape(-1)


def fd_problem(name, shape, coeff, boxes, overlap, *, tau_sharp=None, fixed_k=None, rtol=1e-8, rhs_seed=0):
    n = int(np.prod(shape))
    ro, ci, va = _fd_matrix(shape, coeff)
    owner = _box_owner(shape, boxes)
    omega = overlap_closure(n, ro, ci, owner, int(np.prod(boxes)), overlap)
    b = uniform(rhs_seed, n, -1.0, 1.0)
    return Problem(name, n, ro, ci, va, b, omega, tau_sharp=tau_sharp, fixed_k=fixed_k, rtol=rtol,
                   meta={"shape": list(shape), "boxes": list(boxes), "overlap": overlap})


# ---------------------------------------------------------------------------
# Q1 plane-strain elasticity (element formula of proj/src/fem.cpp:53-97)


def element_stiffness(h: float, e: float, nu: float) -> np.ndarray:
    """8x8 Q1 element stiffness, dof order (ux,uy) per node, nodes
    (0,0),(1,0),(1,1),(0,1); 2x2 Gauss; mirrors the upper triangle."""
    mu = e / (2.0 * (1.0 + nu))
    lam = e * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    d00, d01, d22 = 2.0 * mu + lam, lam, mu
    g = 1.0 / np.sqrt(3.0)
    detj = h * h / 4.0
    ds = 2.0 / h
    ke = np.zeros((8, 8))
    for xi in (-g, g):
        for eta in (-g, g):
            dxi = np.array([-(1 - eta) / 4, (1 - eta) / 4, (1 + eta) / 4, -(1 + eta) / 4]) * ds
            deta = np.array([-(1 - xi) / 4, -(1 + xi) / 4, (1 + xi) / 4, (1 - xi) / 4]) * ds
            for a in range(4):
                for b in range(4):
                    ke[2 * a, 2 * b] += detj * (d00 * dxi[a] * dxi[b] + d22 * deta[a] * deta[b])
                    ke[2 * a, 2 * b + 1] += detj * (d01 * dxi[a] * deta[b] + d22 * deta[a] * dxi[b])
                    ke[2 * a + 1, 2 * b] += detj * (d01 * deta[a] * dxi[b] + d22 * dxi[a] * deta[b])
                    ke[2 * a + 1, 2 * b + 1] += detj * (d00 * deta[a] * deta[b] + d22 * dxi[a] * dxi[b])
    iu = np.triu_indices(8, 1)
    ke[(iu[1], iu[0])] = ke[iu]
    return ke


def elasticity_problem(name, nodes_x, nodes_y, layer_thickness, materials, boxes, overlap, *, tau_sharp=0.1,
                       rtol=1e-8, load=(0.0, -9.81)):
    """Layered Q1 plane strain on a nodes_x x nodes_y mesh (h = 1), the x = 0
    node column clamped (both components eliminated, fem.cpp:111-118).
    Element row ey belongs to layer ey // layer_thickness; layers alternate
    through ``materials`` = [(E, nu), ...] starting at the bottom.  Duplicate
    couplings are summed in element order (TripletBuilder, sparse.cpp:19-47)."""
    nex, ney = nodes_x - 1, nodes_y - 1
    node_dofs = -np.ones((nodes_y, nodes_x, 2), dtype=np.int64)
    free = np.zeros((nodes_y, nodes_x), dtype=bool)
    free[:, 1:] = True
    nfree = int(free.sum())
    node_dofs[free, 0] = 2 * np.arange(nfree)
    node_dofs[free, 1] = 2 * np.arange(nfree) + 1
    n = 2 * nfree
    kes = [element_stiffness(1.0, e, nu) for (e, nu) in materials]
    ey, ex = np.meshgrid(np.arange(ney), np.arange(nex), indexing="ij")
    ey, ex = ey.reshape(-1), ex.reshape(-1)  # element order: ey outer, ex inner
    mat = (ey // layer_thickness) % len(materials)
    nodes = [(ex, ey), (ex + 1, ey), (ex + 1, ey + 1), (ex, ey + 1)]
    dofs = np.stack([node_dofs[y, x, d] for (x, y) in nodes for d in (0, 1)], axis=1)  # (ne, 8)
    kstack = np.stack(kes)[mat]  # (ne, 8, 8)
    la, lb = np.meshgrid(np.arange(8), np.arange(8), indexing="ij")
    r = dofs[:, la.reshape(-1)].reshape(-1)
    c = dofs[:, lb.reshape(-1)].reshape(-1)
    v = kstack[:, la.reshape(-1), lb.reshape(-1)].reshape(-1)
    keep = (r >= 0) & (c >= 0)
    r, c, v = r[keep], c[keep], v[keep]
    order = np.lexsort((c, r))  # stable: duplicates keep insertion order
    r, c, v = r[order], c[order], v[order]
    key = r * n + c
    first = np.ones(key.size, dtype=bool)
    first[1:] = key[1:] != key[:-1]
    starts = np.flatnonzero(first)
    sizes = np.diff(np.append(starts, key.size))
    acc = np.zeros(starts.size)
    for p in range(int(sizes.max())):
        m = sizes > p
        acc[m] = acc[m] + v[starts[m] + p]
    rows_u, cols_u = r[starts], c[starts]
    row_offsets = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_offsets, rows_u + 1, 1)
    row_offsets = np.cumsum(row_offsets)
    # Body force: integral of N_a g, accumulated per element in order.
    g = 1.0 / np.sqrt(3.0)
    bvals = np.zeros(n)
    contrib_rows, contrib_vals = [], []
    for xi in (-g, g):
        for eta in (-g, g):
            shape = [(1 - xi) * (1 - eta) / 4, (1 + xi) * (1 - eta) / 4, (1 + xi) * (1 + eta) / 4,
                     (1 - xi) * (1 + eta) / 4]
            for a in range(4):
                for d in range(2):
                    contrib_rows.append(dofs[:, 2 * a + d])
                    contrib_vals.append(np.full(dofs.shape[0], 0.25 * shape[a] * load[d]))
    cr = np.stack(contrib_rows, axis=1).reshape(-1)  # element-major insertion order
    cv = np.stack(contrib_vals, axis=1).reshape(-1)
    ok = cr >= 0
    cr, cv = cr[ok], cv[ok]
    o = np.argsort(cr, kind="stable")
    cr, cv = cr[o], cv[o]
    st = np.flatnonzero(np.r_[True, cr[1:] != cr[:-1]])
    sz = np.diff(np.append(st, cr.size))
    bacc = np.zeros(st.size)
    for p in range(int(sz.max())):
        m = sz > p
        bacc[m] = bacc[m] + cv[st[m] + p]
    bvals[cr[st]] = bacc
    # Partition: nodal boxes, dofs of free nodes, then algebraic overlap.
    bw, bh = nodes_x // boxes[0], nodes_y // boxes[1]
    iy, ix = np.meshgrid(np.arange(nodes_y), np.arange(nodes_x), indexing="ij")
    node_owner = (ix // bw) + boxes[0] * (iy // bh)
    owner = np.empty(n, dtype=np.int64)
    owner[node_dofs[free, 0]] = node_owner[free]
    owner[node_dofs[free, 1]] = node_owner[free]
    omega = overlap_closure(n, row_offsets.astype(np.int32), cols_u.astype(np.int32), owner,
                            boxes[0] * boxes[1], overlap)
    return Problem(name, n, row_offsets.astype(np.int32), cols_u.astype(np.int32), acc, bvals, omega,
                   tau_sharp=tau_sharp, rtol=rtol,
                   meta={"nodes": [nodes_x, nodes_y], "boxes": list(boxes), "overlap": overlap})


# ---------------------------------------------------------------------------
# The BASELINE.json configurations and small analogues for parity fixtures


def c2_channels(nx, ny, seed=1, band=8, contrast=1e6):
    """Cell coefficient 1e6 on one 1-cell-thick row per 8-row band (row offset
    U{0..7} per band from ``seed``), 1 elsewhere."""
    nb = ny // band
    off = np.floor(uniform01(seed, nb) * band).astype(np.int64)
    c = np.ones((ny, nx))
    for b in range(nb):
        c[b * band + off[b], :] = contrast
    return c.reshape(-1)


def lognormal(n, seed=1, sigma=2.0):
    return np.exp(sigma * normal(seed, n))


def block_powers(shape, block, seed=1, lo=-3.0, hi=3.0):
    """10^U(lo,hi) per block^d cell block (blocks lexicographic, x fastest)."""
    nb = [s // block for s in shape]
    vals = 10.0 ** uniform(seed, int(np.prod(nb)), lo, hi)
    grids = np.meshgrid(*[np.arange(s) for s in reversed(shape)], indexing="ij")
    bidx = np.zeros(grids[0].shape, dtype=np.int64)
    mult = 1
    for ax in range(len(shape)):
        bidx += (grids[len(shape) - 1 - ax] // block) * mult
        mult *= nb[ax]
    return vals[bidx.reshape(-1)]


def spec(name: str) -> dict:
    """Generator arguments of the BASELINE.json configs (c1..c5) and the small
    analogues used for committed parity fixtures: kind "fd" (cell grid) or
    "elasticity" (Q1 mesh).  make() builds them on the host, the GPU-side
    assembly (awg.context_from_spec) on the device."""
    def fd(shape, coeff, boxes, overlap, **kw):
        return dict(kind="fd", name=name, shape=shape, coeff=coeff, boxes=boxes, overlap=overlap, **kw)

    def el(nodes_x, nodes_y, layer, materials, boxes, overlap, **kw):
        return dict(kind="elasticity", name=name, nodes_x=nodes_x, nodes_y=nodes_y, layer_thickness=layer,
                    materials=materials, boxes=boxes, overlap=overlap, **kw)

    soft_hard = [(1e7, 0.45), (1.0, 0.3)]
    if name == "c1":
        return fd((32, 32), np.ones(1024), (2, 2), 1, tau_sharp=0.5)
    if name == "c2":
        return fd((256, 256), c2_channels(256, 256), (4, 4), 2, tau_sharp=0.1)
    if name == "c3":
        return fd((64, 64, 64), lognormal(64 ** 3), (4, 4, 4), 1, fixed_k=10)
    if name == "c4":
        return el(512, 128, 8, soft_hard, (8, 4), 1, tau_sharp=0.1)
    if name == "c5":
        return fd((96, 96, 96), block_powers((96, 96, 96), 8), (6, 6, 6), 1, fixed_k=8)
    # small analogues (same generators, fixture-sized)
    if name == "t2d":  # c1 analogue with n- > 0 via channels
        return fd((24, 24), c2_channels(24, 24, band=6, contrast=1e3), (2, 2), 1, tau_sharp=0.2)
    if name == "t2d_ov2":  # c2 analogue
        return fd((24, 24), c2_channels(24, 24), (2, 2), 2, tau_sharp=0.1)
    if name == "t3d":  # c3 analogue (fixed k)
        return fd((8, 8, 8), lognormal(512), (2, 2, 2), 1, fixed_k=4)
    if name == "t3d_blocks":  # c5 analogue (fixed k)
        return fd((8, 8, 8), block_powers((8, 8, 8), 4), (2, 2, 2), 1, fixed_k=3)
    if name == "telas":  # c4 analogue
        return el(16, 8, 2, soft_hard, (2, 1), 1, tau_sharp=0.1)
    if name == "telas8":  # c4 analogue with c4's 8-element layers and 2x2 nodal boxes
        return el(32, 16, 8, soft_hard, (2, 2), 1, tau_sharp=0.1)
    if name == "tragged":  # ragged boxes (23 x 17 cells in 3 x 2 boxes: 7/7/9 by 8/9), 1 x 1 ... 9 x 9 corner blocks
        return fd((23, 17), c2_channels(23, 17, band=6, contrast=1e3), (3, 2), 1, tau_sharp=0.2)
    if name == "t1box":  # one subdomain: B^s = A, no negative modes, H1 = A^-1
        return fd((12, 12), np.ones(144), (1, 1), 1, tau_sharp=0.5)
    if name == "c4mid":  # c4 with c4-sized subdomains (n_s ~ 4,200) but 4 of them
        return el(128, 64, 8, soft_hard, (2, 2), 1, tau_sharp=0.1)
    if name == "c4s":  # between telas8 and c4mid (n_s ~ 2,400, six 8-element layers)
        return el(96, 48, 8, soft_hard, (2, 2), 1, tau_sharp=0.1)
    raise KeyError(name)


def make(name: str) -> Problem:
    """BASELINE.json configs (c1..c5) and the small analogues (t*), built on
    the host."""
    sp = dict(spec(name))
    kind = sp.pop("kind")
    if kind == "fd":
        return fd_problem(sp.pop("name"), sp.pop("shape"), sp.pop("coeff"), sp.pop("boxes"), sp.pop("overlap"), **sp)
    return elasticity_problem(sp.pop("name"), sp.pop("nodes_x"), sp.pop("nodes_y"), sp.pop("layer_thickness"),
                              sp.pop("materials"), sp.pop("boxes"), sp.pop("overlap"), **sp)


CONFIGS = ["c1", "c2", "c3", "c4", "c5"]
ANALOGUES = ["t2d", "t2d_ov2", "t3d", "t3d_blocks", "telas", "telas8", "tragged", "t1box"]
