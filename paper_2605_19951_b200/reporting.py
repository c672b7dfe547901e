"""Timing/verification helpers of the hot path (rbainv.reporting subset).

Mirrors ``pole_solution_checksum`` (reporting.py:83-84), ``fit_timing_model``
(:63-80), ``scaling_benchmark`` (:87-122) -- the C2 harness template -- and the
run-directory format (``write_run_artifacts`` / ``consolidate_report``,
:125-205: state.json, convergence.csv, timing.csv, residual_heatmap.csv,
transients.csv), which is also the resume point (``load_state`` ->
``InversionConfig.m0``, inversion.py:63,218).  On
the GPU the pole work of one rank is batched into the same launches, so
"workers" are the ranks of the job (G = world size) rather than host threads;
the device path is deterministic, so the checksums are bit-identical for any
worker count exactly as the reference requires.  Multi-source data
([source][channel][receiver]) adds a leading source column to the
per-receiver CSVs.
"""

from __future__ import annotations

import csv
import hashlib
import json
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .shifted import ShiftedFactorCache, resolve_with_cache

__all__ = ["TimingModel", "fit_timing_model", "pole_solution_checksum", "scaling_benchmark",
           "RunReport", "write_run_artifacts", "consolidate_report", "load_state"]


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
    """reporting.py:87-122 on the device.  "Workers" are pole shards (GPU
    ranks): W workers own poles {i : i mod W == r} (PoleWorkerPool,
    shifted.py:147-149).

    * In a multi-process job (torch.distributed initialised, W == world size)
      every rank times its own shard and the row carries the max over ranks.
    * In one process the W shards run one after another on this device, each
      in its own engine; every shard's factorisation and solve times are real
      device times, and the row reports the slowest shard -- the time W GPUs
      running concurrently would take, the all-gather excluded -- with
      ``emulated=True``.

    The pole-solution checksum is taken over all poles in pole order, so it
    must be identical for every W (the reference's worker-count invariance,
    test_acceptance.py:212-234)."""
    import torch
    from .engine import Engine
    from .parallel import PoleComm, ShardComm
    rhs = problem.f if rhs is None else rhs
    rhs = np.asarray(rhs, dtype=complex)
    real = PoleComm.current()
    m = len(approx.poles)
    rows = []
    t1_total = None
    for w in worker_counts:
        w = int(w)
        emulated = real.world == 1
        if not emulated and w != real.world:
            raise ValueError("in a distributed job worker_counts must equal the world size")
        shards = range(w) if emulated else [real.rank]
        g_all = [None] * m
        t_fact = t_solve = 0.0
        for r in shards:
            comm = ShardComm(w, r) if emulated else real
            eng = Engine(problem, approx, comm=comm)
            eng.set_model(model.m)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            torch.cuda.synchronize()
            ev[0].record()
            eng.factor()
            ev[1].record()
            rhs_d = torch.as_tensor(rhs, device=eng.device)
            for _ in range(solve_repeats):
                g = [eng.solve_d(slot, rhs_d) for slot in range(len(eng.local))]
            ev[2].record()
            torch.cuda.synchronize()
            tf, ts = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]) / solve_repeats
            if not emulated:
                t = torch.tensor([tf, ts], dtype=torch.float64, device=eng.device)
                torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                tf, ts = float(t[0]), float(t[1])
                nmax = comm.n_max(m)
                loc = torch.zeros((nmax, eng.N), dtype=torch.complex128, device=eng.device)
                for slot in range(len(eng.local)):
                    loc[slot] = g[slot]
                allg = comm.gather_partials(loc)
                for i, row in enumerate(comm.slot_of_pole(m)):
                    g_all[i] = allg[int(row)].cpu().numpy()
            else:
                for slot, i in enumerate(eng.local):
                    g_all[i] = g[slot].cpu().numpy()
            t_fact = max(t_fact, tf)
            t_solve = max(t_solve, ts)
            eng.close()
        total = t_fact + t_solve
        if t1_total is None and w == 1:
            t1_total = total
        eff = t1_total / (w * total) if (t1_total is not None and total > 0) else np.nan
        rows.append({"workers": w, "factorize_ms": t_fact, "solve_ms": t_solve,
                     "efficiency": eff, "emulated": emulated,
                     "checksum": pole_solution_checksum(np.array(g_all))})
    return rows


# ---------------------------------------------------------------------------
# run directory (reporting.py:125-205)
# ---------------------------------------------------------------------------
CONVERGENCE_FIELDS = ("nu", "phi", "misfit", "reg_value", "chi2", "lam", "eta", "accepted",
                      "lsqr_iters", "lsqr_istop", "wall_ms", "factorizations", "solves",
                      "phi_evals", "phi_before", "directional_slope")


@dataclass
class RunReport:
    iterations: list
    timing: TimingModel | None
    counters: dict
    scaling: list = field(default_factory=list)


def _state_json(state) -> dict:
    return {"model": np.asarray(state.model.m).tolist(),
            "model_ref": np.asarray(state.model.m_ref).tolist(),
            "lambda": float(state.lam), "phi": float(state.phi), "chi2": float(state.chi2),
            "iterations_run": int(state.nu), "diagnostic": state.diagnostic,
            "counters": dict(state.counters),
            "history": [h.as_dict() for h in state.history]}


def _jsonable(v):
    if isinstance(v, (np.floating, np.integer, np.bool_)):
        return v.item()
    raise TypeError(f"not JSON serialisable: {type(v)}")


def write_run_artifacts(rundir, state, data, problem, approx, d_pred) -> None:
    """Persist one inversion run: state.json (model, lambda, objective,
    history, counters), convergence.csv and timing.csv (the history), and the
    per-receiver residual_heatmap.csv (weighted residual per time channel) and
    transients.csv (long format: receiver, time, observed, predicted)."""
    out = Path(rundir)
    out.mkdir(parents=True, exist_ok=True)
    (out / "state.json").write_text(json.dumps(_state_json(state), indent=1, default=_jsonable))
    rows = [h.as_dict() for h in state.history]
    with open(out / "convergence.csv", "w", newline="") as fh:
        wr = csv.DictWriter(fh, fieldnames=list(CONVERGENCE_FIELDS), extrasaction="ignore")
        wr.writeheader()
        wr.writerows(rows)
    with open(out / "timing.csv", "w", newline="") as fh:
        wr = csv.writer(fh)
        wr.writerow(["nu", "lsqr_iters", "wall_ms"])
        for h in state.history:
            wr.writerow([h.nu, h.lsqr_iters, h.wall_ms])
    times = np.asarray(approx.channels.times)
    Kt, Mr = times.size, int(problem.Q.shape[0])
    d_pred = np.asarray(d_pred.cpu().numpy() if hasattr(d_pred, "cpu") else d_pred, dtype=float)
    S = d_pred.size // (Kt * Mr)
    wres = (np.asarray(data.weights) * (d_pred - np.asarray(data.d_obs))).reshape(S, Kt, Mr)
    obs = np.asarray(data.d_obs).reshape(S, Kt, Mr)
    pred = d_pred.reshape(S, Kt, Mr)
    src = ["source"] if S > 1 else []
    with open(out / "residual_heatmap.csv", "w", newline="") as fh:
        wr = csv.writer(fh)
        wr.writerow(src + ["time_s"] + [f"rx{r}" for r in range(Mr)])
        for s_ in range(S):
            for j in range(Kt):
                wr.writerow(([s_] if S > 1 else []) + [times[j]] + wres[s_, j].tolist())
    with open(out / "transients.csv", "w", newline="") as fh:
        wr = csv.writer(fh)
        wr.writerow(src + ["receiver", "time_s", "observed", "predicted"])
        for s_ in range(S):
            for r in range(Mr):
                for j in range(Kt):
                    wr.writerow(([s_] if S > 1 else []) +
                                [r, times[j], obs[s_, j, r], pred[s_, j, r]])


def consolidate_report(rundir) -> RunReport:
    """reporting.py:190-205: the report of a run directory (history, timing
    model when at least 3 iterations ran, counters, optional scaling.json)."""
    out = Path(rundir)
    doc = json.loads((out / "state.json").read_text())
    hist = doc["history"]
    timing = fit_timing_model(hist) if len(hist) >= 3 else None
    scaling = json.loads((out / "scaling.json").read_text()) if (out / "scaling.json").exists() \
        else []
    return RunReport(iterations=hist, timing=timing, counters=doc.get("counters", {}),
                     scaling=scaling)


def load_state(rundir):
    """(m, m_ref, lambda) of a run directory: resume by passing m as
    InversionConfig.m0 and lambda as lambda0 (inversion.py:63,218)."""
    doc = json.loads((Path(rundir) / "state.json").read_text())
    return np.asarray(doc["model"]), np.asarray(doc["model_ref"]), float(doc["lambda"])
