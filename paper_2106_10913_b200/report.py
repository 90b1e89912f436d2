"""Report files of a solve in the reference's formats:

* ``<label>_report.json``   run_with_context (proj/src/harness.cpp:157-218)
* ``<label>_residuals.csv`` write_residual_csv (proj/src/krylov.cpp:161-168)
* ``rows.csv``              TableRow CSV (harness.cpp:47-61, 220-224)

The colorings are the greedy bounds of partition.cpp:120-199 (report-only
quantities; host bookkeeping on the partition)."""
from __future__ import annotations

import json
import os
from typing import List, Optional

import numpy as np


def _memberships(omega, n):
    subs = [[] for _ in range(n)]
    for s, om in enumerate(omega):
        for i in om:
            subs[int(i)].append(s)
    return subs


def _greedy(n_sub, inter):
    color = [-1] * n_sub
    ncol = 0
    for s in range(n_sub):
        used = {color[t] for t in range(s) if inter[s][t]}
        c = 0
        while c in used:
            c += 1
        color[s] = c
        ncol = max(ncol, c + 1)
    return ncol


def coloring_constant(row_offsets, col_indices, omega, n) -> int:
    """partition.cpp:158-170"""
    N = len(omega)
    subs = _memberships(omega, n)
    inter = np.zeros((N, N), dtype=bool)
    for i in range(n):
        for k in range(row_offsets[i], row_offsets[i + 1]):
            j = col_indices[k]
            for s in subs[i]:
                for t in subs[j]:
                    if s != t:
                        inter[s, t] = inter[t, s] = True
    return _greedy(N, inter)


def coloring_constant_aplus(row_offsets, col_indices, omega, n, has_negative) -> int:
    """partition.cpp:172-199"""
    N = len(omega)
    subs = _memberships(omega, n)
    inter = np.zeros((N, N), dtype=bool)
    touches = np.zeros((N, N), dtype=bool)
    for i in range(n):
        for k in range(row_offsets[i], row_offsets[i + 1]):
            j = col_indices[k]
            for s in subs[i]:
                for t in subs[j]:
                    if s != t:
                        inter[s, t] = inter[t, s] = True
        for s in subs[i]:
            for t in subs[i]:
                touches[s, t] = True
    for u in range(N):
        if not has_negative[u]:
            continue
        for s in range(N):
            if not touches[u, s]:
                continue
            for t in range(N):
                if touches[u, t] and s != t:
                    inter[s, t] = inter[t, s] = True
    return _greedy(N, inter)


def table_row(label, rep, n0, n_minus) -> dict:
    return {"label": label, "kappa": rep.kappa_estimate, "it": rep.iterations, "lambda_min": rep.ritz_min,
            "lambda_max": rep.ritz_max, "v0": n0, "n_minus": n_minus, "converged": rep.converged}


def _fmt(v: float) -> str:
    return "%.6g" % v


def write_outputs(out_dir: str, label: str, ctx, cfg, rep, rtol: float, maxit: int, colorings: bool = True) -> dict:
    """Write the report JSON, residual CSV and the rows.csv line of one solve."""
    os.makedirs(out_dir, exist_ok=True)
    stem = os.path.join(out_dir, "".join(ch if ch.isalnum() else "_" for ch in label))
    with open(stem + "_residuals.csv", "w") as fh:
        fh.write("iteration,relative_residual\n")
        for i, r in enumerate(rep.residual_history):
            fh.write(f"{i + 1},{r:.12g}\n")
    q = ctx.query()
    m = ctx.get("n_nonpos")
    z = ctx.get("n_zero")
    omega = ctx.partition.omega
    a = ctx.a
    n_s_minus = [int(x) for x in (m - z)]
    prob = {"kind": "external", "n": a.n, "nnz": a.nnz, "subdomains": len(omega),
            "subdomain_sizes": [int(len(o)) for o in omega], "n_s_minus": n_s_minus}
    if colorings:
        prob["coloring_A"] = coloring_constant(a.row_offsets, a.col_indices, omega, a.n)
        prob["coloring_Aplus"] = coloring_constant_aplus(a.row_offsets, a.col_indices, omega, a.n,
                                                         [x > 0 for x in n_s_minus])
    one = {0: "AS", 1: "AS_PLUS", 2: "NN"}[int(cfg.one_level)]
    prec = {"one_level": one, "composition": "additive" if int(cfg.composition) == 0 else "hybrid",
            "use_coarse": bool(cfg.use_coarse), "tau_sharp": cfg.tau_sharp, "tau_flat": cfg.tau_flat,
            "awg": ["none", "ad", "hyb", "inex"][int(cfg.awg)], "coarse_dim": q["n0"], "coarse_retained": q["r0"]}
    if int(cfg.awg) != 0:
        prec.update({"w_rtol": cfg.w_rtol, "n_minus": q["n_minus"],
                     "w_inner_iterations": [int(v) for v in ctx.get("w_inner_iterations")], "kw_retained": q["rw"]})
    solve = {"rtol": rtol, "maxit": maxit, "iterations": rep.iterations, "converged": rep.converged,
             "kappa": rep.kappa_estimate, "lambda_min": rep.ritz_min, "lambda_max": rep.ritz_max,
             "final_relative_residual": rep.final_relative_residual,
             "recurrence_residual_at_exit": rep.recurrence_residual_at_exit}
    report = {"label": label, "problem": prob, "preconditioner": prec, "solve": solve}
    with open(stem + "_report.json", "w") as fh:
        json.dump(report, fh, indent=2)
        fh.write("\n")
    row = table_row(label, rep, q["n0"], q["n_minus"] if int(cfg.awg) != 0 else 0)
    rows = os.path.join(out_dir, "rows.csv")
    fresh = not os.path.exists(rows)
    with open(rows, "a") as fh:
        if fresh:
            fh.write("label,kappa,it,lambda_min,lambda_max,v0,n_minus\n")
        fh.write(f"{label},{_fmt(row['kappa'])},{row['it']},{_fmt(row['lambda_min'])},{_fmt(row['lambda_max'])},"
                 f"{row['v0']},{row['n_minus']}\n")
    return report
