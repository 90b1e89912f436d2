"""Python mirror of the reference's proj/include/awg API over the C ABI.

Names, argument meaning and error behaviour follow the reference:

* ``SparseSymMatrix`` / ``Partition``        include/awg/sparse.hpp:12-21, partition.hpp:14-22
* ``PreconditionerConfig`` + enums          include/awg/preconditioner.hpp:17-31
* ``ProblemContext``                        include/awg/harness.hpp:73-98 (owns the device context)
* ``Splitting.apply_Aplus/apply_Aminus``    include/awg/splitting.hpp:51-55
* ``OneLevel`` / ``TwoLevel`` / ``AwgPreconditioner`` ``.apply``   preconditioner.hpp:33-100
* ``coarse_correct``                        include/awg/coarse.hpp:72
* ``pcg`` / ``SolveReport``                 include/awg/krylov.hpp:14-36
* exceptions: ``NotSpdError`` (pivot_index), ``RuntimeError`` (breakdown, non-convergence,
  overlap), ``ValueError`` (std::invalid_argument)

Everything computes on the GPU through ``libawg_b200.so``; there is no CPU
fallback: importing works without a GPU, but creating a context without one
raises.
"""
from __future__ import annotations

import ctypes
import dataclasses
import enum
import os
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libawg_b200.so")

# ---------------------------------------------------------------------------
# enums / config


class OneLevelKind(enum.IntEnum):
    AS = 0
    AS_PLUS = 1
    NN = 2


class Composition(enum.IntEnum):
    ADDITIVE = 0
    HYBRID = 1


class AwgMode(enum.IntEnum):
    NONE = 0
    AD = 1
    HYB = 2
    INEX = 3


class Op(enum.IntEnum):
    A = 0
    AMINUS = 1
    APLUS = 2
    H1 = 3
    Q = 4
    QW = 5
    H2 = 6
    H3 = 7
    PI3 = 8
    PI3T = 9


AWG_OK, AWG_E_ARG, AWG_E_CUDA, AWG_E_NOT_SPD, AWG_E_BREAKDOWN, AWG_E_NO_CONVERGENCE, AWG_E_OVERLAP, AWG_E_STATE = range(8)


class NotSpdError(RuntimeError):
    """include/awg/dense.hpp:58-63"""

    def __init__(self, msg: str, pivot_index: int):
        super().__init__(msg)
        self.pivot_index = pivot_index


class AwgCudaError(RuntimeError):
    pass


@dataclasses.dataclass
class PreconditionerConfig:
    """include/awg/preconditioner.hpp:21-31 defaults, plus the fixed-k rule
     and the rank-revealing-factor semantics switch."""

    one_level: OneLevelKind = OneLevelKind.NN
    composition: Composition = Composition.HYBRID
    use_coarse: bool = True
    tau_sharp: float = 0.1
    tau_flat: float = 10.0
    awg: AwgMode = AwgMode.AD
    w_rtol: float = 1e-10
    fixed_k: int = 0
    rrf_semantics: str = "reference"  # or "exact"
    lu_semantics: str = "reference"  # INEX core solve
    w_maxit_factor: int = 10


@dataclasses.dataclass
class SolveReport:
    """include/awg/krylov.hpp:14-28"""

    iterations: int = 0
    converged: bool = False
    residual_history: List[float] = dataclasses.field(default_factory=list)
    final_relative_residual: float = 0.0
    recurrence_residual_at_exit: float = 0.0
    lanczos_diag: List[float] = dataclasses.field(default_factory=list)
    lanczos_offdiag: List[float] = dataclasses.field(default_factory=list)
    ritz_min: float = 0.0
    ritz_max: float = 0.0
    kappa_estimate: float = 0.0
    solve_ms: float = 0.0


# ---------------------------------------------------------------------------
# ctypes layer


class _Config(ctypes.Structure):
    _fields_ = [
        ("one_level", ctypes.c_int), ("composition", ctypes.c_int), ("use_coarse", ctypes.c_int),
        ("tau_sharp", ctypes.c_double), ("tau_flat", ctypes.c_double), ("fixed_k", ctypes.c_int),
        ("awg_mode", ctypes.c_int), ("w_rtol", ctypes.c_double), ("w_maxit_factor", ctypes.c_int),
        ("rrf_semantics", ctypes.c_int), ("lu_semantics", ctypes.c_int),
    ]


_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


class _Factors(ctypes.Structure):
    _fields_ = [
        ("lam", _dp), ("V", _dp), ("n_nonpos", _ip), ("n_zero", _ip), ("ks", _ip), ("Y", _dp),
        ("r0", ctypes.c_int), ("k0_retained", _ip), ("k0_l11", _dp),
        ("n_minus", ctypes.c_int), ("W", _dp), ("neg_weights", _dp), ("v_minus", _dp),
        ("rw", ctypes.c_int), ("kw_retained", _ip), ("kw_l11", _dp),
    ]


class _Report(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int), ("converged", ctypes.c_int),
        ("final_relative_residual", ctypes.c_double), ("recurrence_residual_at_exit", ctypes.c_double),
        ("ritz_min", ctypes.c_double), ("ritz_max", ctypes.c_double), ("kappa_estimate", ctypes.c_double),
        ("solve_ms", ctypes.c_double),
    ]


class _Stats(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int), ("nnz", ctypes.c_int), ("n_sub", ctypes.c_int), ("n0", ctypes.c_int),
        ("r0", ctypes.c_int), ("n_minus", ctypes.c_int), ("rw", ctypes.c_int),
        ("sum_ns", ctypes.c_longlong), ("sum_ns2", ctypes.c_longlong), ("sum_ns_ks", ctypes.c_longlong),
        ("sum_ns_ms", ctypes.c_longlong), ("sum_ns_qs", ctypes.c_longlong),
        ("t_setup_ms", ctypes.c_double * 8), ("w_inner_total", ctypes.c_int), ("w_batches", ctypes.c_int),
        ("nn_single_pass", ctypes.c_int), ("nn_static_split", ctypes.c_int), ("coarse_az", ctypes.c_int),
    ]


EXPORTED_SYMBOLS = [
    "awg_create", "awg_destroy", "awg_last_error", "awg_last_error_index", "awg_set_matrix",
    "awg_set_partition", "awg_setup", "awg_load_factors", "awg_apply", "awg_pcg", "awg_query",
    "awg_get_history", "awg_get_array", "awg_launch_count", "awg_time_apply", "awg_time_kernel",
    "awg_synthetic_factors", "awg_kernel_timer", "awg_assemble_fd", "awg_assemble_elasticity", "awg_partition_owner",
    "awg_partition_boxes", "awg_bench_dgemm", "awg_set_option", "awg_pivoted_factor",
    "awg_coarse_solve", "awg_bench_eig",
]

_lib = None


def load_library(path: str = LIB_PATH):
    """Load the CUDA library; fails loudly (no fallback) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    vp = ctypes.c_void_p
    lib.awg_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int]
    lib.awg_destroy.argtypes = [vp]
    lib.awg_destroy.restype = None
    lib.awg_last_error.argtypes = [vp]
    lib.awg_last_error.restype = ctypes.c_char_p
    lib.awg_last_error_index.argtypes = [vp]
    lib.awg_set_matrix.argtypes = [vp, ctypes.c_int, _ip, _ip, _dp]
    lib.awg_set_partition.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_longlong), _ip]
    lib.awg_assemble_fd.argtypes = [vp, ctypes.c_int, _ip, _dp]
    lib.awg_kernel_timer.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(ctypes.c_longlong)]
    lib.awg_assemble_elasticity.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp, _dp]
    lib.awg_partition_owner.argtypes = [vp, _ip, ctypes.c_int, ctypes.c_int]
    lib.awg_partition_boxes.argtypes = [vp, _ip, ctypes.c_int]
    lib.awg_set_option.argtypes = [vp, ctypes.c_char_p, ctypes.c_longlong]
    lib.awg_bench_eig.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong, _dp]
    lib.awg_coarse_solve.argtypes = [vp, ctypes.c_int, _dp, _dp]
    lib.awg_pivoted_factor.argtypes = [vp, ctypes.c_int, _dp, ctypes.c_int, _ip, _ip, _dp]
    lib.awg_setup.argtypes = [vp, ctypes.POINTER(_Config)]
    lib.awg_load_factors.argtypes = [vp, ctypes.POINTER(_Config), ctypes.POINTER(_Factors)]
    lib.awg_apply.argtypes = [vp, ctypes.c_int, vp, vp, ctypes.c_int]
    lib.awg_pcg.argtypes = [vp, vp, vp, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_Report)]
    lib.awg_query.argtypes = [vp, ctypes.POINTER(_Stats)]
    lib.awg_get_history.argtypes = [vp, ctypes.c_int, _dp, ctypes.c_int]
    lib.awg_get_array.argtypes = [vp, ctypes.c_int, vp, ctypes.c_longlong, ctypes.POINTER(ctypes.c_longlong)]
    lib.awg_launch_count.argtypes = [vp]
    lib.awg_launch_count.restype = ctypes.c_longlong
    lib.awg_time_apply.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    lib.awg_time_kernel.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_double)]
    lib.awg_synthetic_factors.argtypes = [vp, ctypes.c_int, ctypes.c_ulonglong]
    lib.awg_bench_dgemm.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    _lib = lib
    return lib


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


# ---------------------------------------------------------------------------
# problem containers


@dataclasses.dataclass
class SparseSymMatrix:
    """CSR with both triangles stored (sparse.hpp:12-21)."""

    n: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(len(self.col_indices))


@dataclasses.dataclass
class Partition:
    """omega[s]: sorted, duplicate-free global dofs (partition.hpp:14-22)."""

    omega: List[np.ndarray]
    n: int

    def count(self) -> int:
        return len(self.omega)

    def size_of(self, s: int) -> int:
        return int(len(self.omega[s]))


_ARRAYS = {"lam": (0, "f"), "n_nonpos": (1, "i"), "n_zero": (2, "i"), "ks": (3, "i"), "pencil_lam": (4, "f"),
           "multiplicity": (5, "i"), "k0_retained": (6, "i"), "k0_l11": (7, "f"), "kw_retained": (8, "i"),
           "kw_l11": (9, "f"), "W": (10, "f"), "neg_weights": (11, "f"), "w_inner_iterations": (12, "i"),
           "Y": (13, "f"), "V": (14, "f"), "eps_zero": (15, "f"), "assembled_rhs": (16, "f"),
           "row_offsets": (17, "i"), "col_indices": (18, "i"), "values": (19, "f"), "part_offsets": (20, "i"),
           "part_indices": (21, "i")}


class ProblemContext:
    """Owns one device context: the system, the partition and every setup
    product (ProblemContext, harness.hpp:73-98).  ``setup(cfg)`` builds the
    preconditioner on the GPU; ``load_factors`` takes them from an external
    factorization (the apply-parity protocol)."""

    def __init__(self, a: SparseSymMatrix, b: Optional[np.ndarray], partition: Partition, device: int = 0):
        self._lib = load_library()
        h = ctypes.c_void_p()
        rc = self._lib.awg_create(ctypes.byref(h), device)
        self._h = h
        if rc != AWG_OK:
            msg = self._lib.awg_last_error(h).decode()
            self._lib.awg_destroy(h)
            self._h = None
            raise AwgCudaError(msg)
        self.a = a
        self.b = None if b is None else _f64(b)
        self.partition = partition
        if b is not None and len(b) != a.n:
            raise RuntimeError("external problem: rhs size does not match matrix")
        self._keep = [_i32(a.row_offsets), _i32(a.col_indices), _f64(a.values)]
        self._check(self._lib.awg_set_matrix(self._h, a.n, _ptr(self._keep[0], ctypes.c_int),
                                              _ptr(self._keep[1], ctypes.c_int), _ptr(self._keep[2], ctypes.c_double)))
        off = np.zeros(partition.count() + 1, dtype=np.int64)
        off[1:] = np.cumsum([len(o) for o in partition.omega])
        idx = _i32(np.concatenate(partition.omega)) if partition.count() else np.zeros(0, np.int32)
        self._check(self._lib.awg_set_partition(self._h, partition.count(), _ptr(off, ctypes.c_longlong),
                                                 _ptr(idx, ctypes.c_int)))
        self.cfg: Optional[PreconditionerConfig] = None

    # -- GPU-side assembly -------------------------------------
    @classmethod
    def _bare(cls, device: int = 0) -> "ProblemContext":
        self = cls.__new__(cls)
        self._lib = load_library()
        h = ctypes.c_void_p()
        rc = self._lib.awg_create(ctypes.byref(h), device)
        self._h = h
        if rc != AWG_OK:
            msg = self._lib.awg_last_error(h).decode()
            self._lib.awg_destroy(h)
            self._h = None
            raise AwgCudaError(msg)
        self.cfg = None
        self._keep = []
        return self

    def _adopt(self, b) -> None:
        """Host views of the device-assembled system (reports, checks)."""
        n = self.query()["n"]
        self.a = SparseSymMatrix(n, self.get("row_offsets"), self.get("col_indices"), self.get("values"))
        off, idx = self.get("part_offsets"), self.get("part_indices")
        self.partition = Partition([idx[off[s]:off[s + 1]] for s in range(len(off) - 1)], n)
        self.b = None if b is None else _f64(b)

    @classmethod
    def assemble_fd(cls, shape, cell_coef, b, boxes, overlap: int, device: int = 0) -> "ProblemContext":
        """Cell-centred diffusion assembled on the device, box partition with
        ``overlap`` rings of closure computed on the device."""
        self = cls._bare(device)
        sh = _i32(np.asarray(shape))
        coef = _f64(cell_coef)
        self._check(self._lib.awg_assemble_fd(self._h, len(sh), _ptr(sh, ctypes.c_int), _ptr(coef, ctypes.c_double)))
        bx = _i32(np.asarray(boxes))
        self._check(self._lib.awg_partition_boxes(self._h, _ptr(bx, ctypes.c_int), int(overlap)))
        self._adopt(b)
        return self

    @classmethod
    def assemble_elasticity(cls, nodes_x: int, nodes_y: int, layer_thickness: int, materials, boxes, overlap: int,
                            load=(0.0, -9.81), device: int = 0) -> "ProblemContext":
        """Q1 plane strain assembled on the device (fem.cpp:99-162 rules); the
        body-force rhs comes back from the device."""
        self = cls._bare(device)
        e = _f64([m[0] for m in materials])
        nu = _f64([m[1] for m in materials])
        ld = _f64(load)
        self._check(self._lib.awg_assemble_elasticity(self._h, int(nodes_x), int(nodes_y), int(layer_thickness),
                                                       len(e), _ptr(e, ctypes.c_double), _ptr(nu, ctypes.c_double),
                                                       _ptr(ld, ctypes.c_double)))
        bx = _i32(np.asarray(boxes))
        self._check(self._lib.awg_partition_boxes(self._h, _ptr(bx, ctypes.c_int), int(overlap)))
        self._adopt(self.get("assembled_rhs"))
        return self

    # -- plumbing ------------------------------------------------------------
    def _check(self, rc: int):
        if rc == AWG_OK:
            return
        msg = self._lib.awg_last_error(self._h).decode()
        if rc == AWG_E_NOT_SPD:
            raise NotSpdError(msg, int(self._lib.awg_last_error_index(self._h)))
        if rc == AWG_E_ARG:
            raise ValueError(msg)
        if rc == AWG_E_CUDA:
            raise AwgCudaError(msg)
        raise RuntimeError(msg)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.awg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _cfg(cfg: PreconditionerConfig) -> _Config:
        return _Config(int(cfg.one_level), int(cfg.composition), int(bool(cfg.use_coarse)), float(cfg.tau_sharp),
                       float(cfg.tau_flat), int(cfg.fixed_k), int(cfg.awg), float(cfg.w_rtol),
                       int(cfg.w_maxit_factor), 0 if cfg.rrf_semantics == "reference" else 1,
                       0 if cfg.lu_semantics == "reference" else 1)

    # -- setup -----------------------------------------------------------------
    def setup(self, cfg: PreconditionerConfig):
        c = self._cfg(cfg)
        self._check(self._lib.awg_setup(self._h, ctypes.byref(c)))
        self.cfg = cfg

    def load_factors(self, cfg: PreconditionerConfig, f: Dict[str, np.ndarray]):
        """Setup products as exported by the oracle driver (see tests/golden)."""
        keep = {}

        def d(name):
            if name not in f or f[name] is None:
                return None
            keep[name] = _f64(np.asarray(f[name]).reshape(-1, order="F"))
            return _ptr(keep[name], ctypes.c_double)

        def i(name):
            if name not in f or f[name] is None:
                return None
            keep[name] = _i32(np.asarray(f[name]).reshape(-1))
            return _ptr(keep[name], ctypes.c_int)

        fac = _Factors()
        fac.lam, fac.V, fac.n_nonpos, fac.n_zero, fac.ks, fac.Y = d("lam"), d("V"), i("n_nonpos"), i("n_zero"), i("ks"), d("Y")
        fac.r0 = int(len(f["k0_retained"])) if "k0_retained" in f else 0
        fac.k0_retained, fac.k0_l11 = i("k0_retained"), d("k0_l11")
        fac.n_minus = int(np.asarray(f["W"]).shape[1]) if "W" in f and f["W"] is not None else 0
        fac.W, fac.neg_weights, fac.v_minus = d("W"), d("neg_weights"), d("v_minus")
        fac.rw = int(len(f["kw_retained"])) if "kw_retained" in f else 0
        fac.kw_retained, fac.kw_l11 = i("kw_retained"), d("kw_l11")
        c = self._cfg(cfg)
        self._check(self._lib.awg_load_factors(self._h, ctypes.byref(c), ctypes.byref(fac)))
        self.cfg = cfg

    # -- operators -------------------------------------------------------------
    def apply(self, op: Op, x):
        """y = op x.  numpy in -> numpy out (host pointers, copies inside);
        torch CUDA tensor in -> torch CUDA tensor out (device pointers)."""
        if hasattr(x, "is_cuda") and x.is_cuda:
            import torch

            xx = x.contiguous().to(torch.float64)
            y = torch.empty_like(xx)
            torch.cuda.current_stream().synchronize()
            self._check(self._lib.awg_apply(self._h, int(op), ctypes.c_void_p(xx.data_ptr()),
                                             ctypes.c_void_p(y.data_ptr()), 1))
            return y
        xx = _f64(x)
        if xx.shape != (self.a.n,):
            raise ValueError("apply: dimension mismatch")
        y = np.empty_like(xx)
        self._check(self._lib.awg_apply(self._h, int(op), xx.ctypes.data_as(ctypes.c_void_p),
                                         y.ctypes.data_as(ctypes.c_void_p), 0))
        return y

    def time_apply(self, op: Op, reps: int = 10) -> float:
        ms = ctypes.c_double()
        self._check(self._lib.awg_time_apply(self._h, int(op), reps, ctypes.byref(ms)))
        return ms.value

    KERNELS = {"nn_gemvT": 0, "nn_gemv": 1, "spmv": 2, "w_gemvT": 3, "w_gemv": 4, "nn_fused": 5}

    def kernel_timer(self, reset: bool = False) -> Tuple[float, int]:
        """(total ms, launches) of the single-pass local solve measured inside
        the kernel since the last reset (covers graph-launched solves)."""
        ms, n = ctypes.c_double(), ctypes.c_longlong()
        self._check(self._lib.awg_kernel_timer(self._h, int(reset), ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def time_kernel(self, name: str, reps: int = 10) -> Tuple[float, float]:
        """(ms per launch, algorithmic bytes per launch) of one hot kernel."""
        ms, by = ctypes.c_double(), ctypes.c_double()
        self._check(self._lib.awg_time_kernel(self._h, self.KERNELS[name], reps, ctypes.byref(ms), ctypes.byref(by)))
        return ms.value, by.value

    def bench_dgemm(self, m: int, n: int, k: int, count: int = 1, reps: int = 5, transpose_a: bool = False) -> dict:
        """Grouped FP64 tensor-core GEMM (the W build's block one-level products)
        against cuBLAS on seeded operands: relative max error, ms, TFLOP/s."""
        out = (ctypes.c_double * 5)()
        self._check(self._lib.awg_bench_dgemm(self._h, m, n, k, count, int(transpose_a), reps, out))
        return {"rel_err": out[0], "ms_grouped": out[1], "ms_cublas": out[2], "tflops_grouped": out[3],
                "tflops_cublas": out[4]}

    def pcg(self, b=None, rtol: float = 1e-10, maxit: int = 10000) -> Tuple[np.ndarray, SolveReport]:
        """pcg(spmv, H3.apply, b, rtol, maxit) — krylov.cpp:36-124, on device."""
        bb = self.b if b is None else _f64(b)
        x = np.empty_like(bb)
        rep = _Report()
        self._check(self._lib.awg_pcg(self._h, bb.ctypes.data_as(ctypes.c_void_p), x.ctypes.data_as(ctypes.c_void_p),
                                       float(rtol), int(maxit), 0, ctypes.byref(rep)))
        out = SolveReport(iterations=rep.iterations, converged=bool(rep.converged),
                          final_relative_residual=rep.final_relative_residual,
                          recurrence_residual_at_exit=rep.recurrence_residual_at_exit, ritz_min=rep.ritz_min,
                          ritz_max=rep.ritz_max, kappa_estimate=rep.kappa_estimate, solve_ms=rep.solve_ms)
        out.residual_history = self._history(0)
        out.lanczos_diag = self._history(1)
        out.lanczos_offdiag = self._history(2)
        return x, out

    def _history(self, which: int) -> List[float]:
        k = self._lib.awg_get_history(self._h, which, None, 0)
        buf = np.zeros(max(k, 1))
        self._lib.awg_get_history(self._h, which, _ptr(buf, ctypes.c_double), k)
        return buf[:k].tolist()

    def query(self) -> dict:
        st = _Stats()
        self._check(self._lib.awg_query(self._h, ctypes.byref(st)))
        out = {name: getattr(st, name) for name, _ in _Stats._fields_ if name != "t_setup_ms"}
        out["t_setup_ms"] = list(st.t_setup_ms)
        return out

    def get(self, name: str) -> np.ndarray:
        which, kind = _ARRAYS[name]
        cnt = ctypes.c_longlong()
        self._check(self._lib.awg_get_array(self._h, which, None, 0, ctypes.byref(cnt)))
        arr = np.empty(max(cnt.value, 1), dtype=np.int32 if kind == "i" else np.float64)
        self._check(self._lib.awg_get_array(self._h, which, arr.ctypes.data_as(ctypes.c_void_p), cnt.value,
                                             ctypes.byref(cnt)))
        return arr[:cnt.value]

    def synthetic_factors(self, m_per_sub: int = 0, seed: int = 1):
        """Benchmark hook: random local factors at full scale (no setup)."""
        self._check(self._lib.awg_synthetic_factors(self._h, int(m_per_sub), int(seed)))

    def launch_count(self) -> int:
        return int(self._lib.awg_launch_count(self._h))

    def coarse_solve(self, which: str, b) -> np.ndarray:
        """rank_revealing_solve (dense.cpp:348-366) with the device's K0
        (which="k0") or KW ("kw") factor."""
        b = _f64(b)
        x = np.zeros_like(b)
        self._check(self._lib.awg_coarse_solve(self._h, 0 if which == "k0" else 1, b.ctypes.data_as(_dp),
                                               x.ctypes.data_as(_dp)))
        return x

    def set_option(self, name: str, value: int) -> "ProblemContext":
        """Experiment switch (tests / profiles only; awg_set_option): the
        product defaults are frozen in the library."""
        self._check(self._lib.awg_set_option(self._h, name.encode(), int(value)))
        return self

    def set_options(self, opts: Optional[Dict[str, int]]) -> "ProblemContext":
        for k, v in (opts or {}).items():
            self.set_option(k, v)
        return self

    # -- reference-shaped views -------------------------------------------------
    def splitting(self) -> "Splitting":
        return Splitting(self)


class Splitting:
    """A+ / A- applies (splitting.hpp:51-55)."""

    def __init__(self, ctx: ProblemContext):
        self.ctx = ctx

    def apply_Aplus(self, x):
        return self.ctx.apply(Op.APLUS, x)

    def apply_Aminus(self, x):
        return self.ctx.apply(Op.AMINUS, x)


class OneLevel:
    def __init__(self, ctx: ProblemContext):
        self.ctx = ctx

    def apply(self, x):
        return self.ctx.apply(Op.H1, x)


class TwoLevel:
    def __init__(self, ctx: ProblemContext):
        self.ctx = ctx

    def apply(self, x):
        return self.ctx.apply(Op.H2, x)


class AwgPreconditioner:
    def __init__(self, ctx: ProblemContext):
        self.ctx = ctx

    def apply(self, x):
        return self.ctx.apply(Op.H3, x)

    def apply_pi3(self, x):
        return self.ctx.apply(Op.PI3, x)

    def apply_pi3_transpose(self, x):
        return self.ctx.apply(Op.PI3T, x)


def coarse_correct(ctx: ProblemContext, x):
    return ctx.apply(Op.Q, x)


def spmv(ctx: ProblemContext, x):
    return ctx.apply(Op.A, x)


def pcg(ctx: ProblemContext, b, rtol: float, maxit: int):
    return ctx.pcg(b, rtol, maxit)


def bench_eig(n: int, count: int = 1, kind: int = 0, seed: int = 1, device: int = 0, verbose: int = 0,
              options: Optional[Dict[str, int]] = None) -> dict:
    """The setup eigensolver (eig.cu) on seeded matrices against cuSOLVER
    (awg_bench_eig): eigenvalue error, residual, orthogonality, timings."""
    ctx = ProblemContext._bare(device)
    try:
        if verbose:
            ctx.set_option("verbose", verbose)
        ctx.set_options(options)
        out = (ctypes.c_double * 5)()
        ctx._check(ctx._lib.awg_bench_eig(ctx._h, int(n), int(count), int(kind), int(seed), out))
        return {"eig_err": out[0], "resid": out[1], "orth": out[2], "ms": out[3], "ms_cusolver": out[4]}
    finally:
        ctx.close()


def pivoted_factor(g, exact: bool = False, device: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """rank_revealing_sym_factor (dense.cpp:299-346) of a symmetric matrix on
    the device (awg_pivoted_factor): (retained pivot order, l11 r x r lower)."""
    g = np.asfortranarray(np.asarray(g, dtype=np.float64))
    n = g.shape[0]
    ctx = ProblemContext._bare(device)
    try:
        rank = ctypes.c_int()
        ret = np.zeros(max(n, 1), dtype=np.int32)
        l11 = np.zeros(max(n * n, 1), dtype=np.float64)
        ctx._check(ctx._lib.awg_pivoted_factor(ctx._h, n, g.ctypes.data_as(_dp), int(bool(exact)), ctypes.byref(rank),
                                               ret.ctypes.data_as(_ip), l11.ctypes.data_as(_dp)))
        r = rank.value
        return ret[:r].copy(), l11[:r * r].reshape(r, r, order="F").copy()
    finally:
        ctx.close()


def context_from_problem(p, device: int = 0, options: Optional[Dict[str, int]] = None) -> ProblemContext:
    """ProblemContext from a problems.Problem (``options``: awg_set_option
    switches, tests / profiles only)."""
    a = SparseSymMatrix(p.n, p.row_offsets, p.col_indices, p.values)
    return ProblemContext(a, p.b, Partition(list(p.omega), p.n), device=device).set_options(options)


def context_from_spec(sp: dict, device: int = 0) -> ProblemContext:
    """ProblemContext assembled on the device from problems.spec(name)."""
    from . import problems

    if sp["kind"] == "fd":
        n = int(np.prod(sp["shape"]))
        b = problems.uniform(0, n, -1.0, 1.0)
        return ProblemContext.assemble_fd(sp["shape"], sp["coeff"], b, sp["boxes"], sp["overlap"], device=device)
    return ProblemContext.assemble_elasticity(sp["nodes_x"], sp["nodes_y"], sp["layer_thickness"], sp["materials"],
                                              sp["boxes"], sp["overlap"], device=device)


def config_for(p, **kw) -> PreconditionerConfig:
    """Reference-default preconditioner (NN, hybrid, AD, w_rtol 1e-10) with
    the problem's selection rule."""
    cfg = PreconditionerConfig(**kw)
    if p.fixed_k:
        cfg.fixed_k = int(p.fixed_k)
    elif p.tau_sharp is not None:
        cfg.tau_sharp = float(p.tau_sharp)
    return cfg
