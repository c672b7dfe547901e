"""Timing/verification helpers of the hot path (rbainv.reporting subset).

Mirrors ``pole_solution_checksum`` (reporting.py:83-84), ``fit_timing_model``
(:63-80) and ``scaling_benchmark`` (:87-122) -- the C2 harness template.  On
the GPU the pole work of one rank is batched into the same launches, so
"workers" are the ranks of the job (G = world size) rather than host threads;
the device path is deterministic, so the checksums are bit-identical for any
worker count exactly as the reference requires.  Rundir/report writers are
out of scope.
"""

from __future__ import annotations

import hashlib
import time
from dataclasses import dataclass

import numpy as np

from .shifted import ShiftedFactorCache, resolve_with_cache

__all__ = ["TimingModel", "fit_timing_model", "pole_solution_checksum", "scaling_benchmark"]


@dataclass
class TimingModel:
    intercept: float
    slope: float
    r_squared: float
    defined: bool = True


def fit_timing_model(history) -> TimingModel:
    """OLS of per-iteration wall time against LSQR iterations (reporting.py:63-80)."""
    rows = [(r.lsqr_iters, r.wall_ms) if hasattr(r, "lsqr_iters")
            else (r["lsqr_iters"], r["wall_ms"]) for r in history]
    if len(rows) < 3:
        raise ValueError("need at least 3 iterations to fit a timing model")
    x = np.array([r[0] for r in rows], dtype=float)
    y = np.array([r[1] for r in rows], dtype=float)
    if np.all(x == x[0]):
        return TimingModel(intercept=float(np.mean(y)), slope=np.nan, r_squared=np.nan,
                           defined=False)
    slope, intercept = np.polyfit(x, y, 1)
    resid = y - (intercept + slope * x)
    ss_tot = float(np.sum((y - y.mean()) ** 2))
    r2 = 1.0 if ss_tot == 0 else 1.0 - float(np.sum(resid ** 2)) / ss_tot
    return TimingModel(intercept=float(intercept), slope=float(slope), r_squared=r2,
                       defined=True)


def pole_solution_checksum(g: np.ndarray) -> str:
    """reporting.py:83-84"""
    return hashlib.sha256(np.ascontiguousarray(g).tobytes()).hexdigest()


def scaling_benchmark(problem, model, approx, worker_counts=(1,), rhs=None,
                      solve_repeats: int = 4) -> list[dict]:
    """Factorise-all and solve-all timings (device events) per repetition of
    `worker_counts`; pole solutions checksummed (reporting.py:87-122)."""
    import torch
    rhs = problem.f if rhs is None else rhs
    rows = []
    t1_total = None
    for w in worker_counts:
        cache = ShiftedFactorCache()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cache.ensure_factored(problem, model, approx)
        torch.cuda.synchronize()
        t_fact = time.perf_counter() - t0
        t0 = time.perf_counter()
        for _ in range(solve_repeats):
            g = np.array([resolve_with_cache(cache, i, rhs) for i in cache.engine.local])
        torch.cuda.synchronize()
        t_solve = (time.perf_counter() - t0) / solve_repeats
        total = t_fact + t_solve
        if t1_total is None:
            t1_total = total
        rows.append({"workers": int(w), "factorize_ms": t_fact * 1e3, "solve_ms": t_solve * 1e3,
                     "efficiency": t1_total / (w * total) if total > 0 else np.nan,
                     "checksum": pole_solution_checksum(g)})
        cache.engine.close()
    return rows
