#!/usr/bin/env python
"""Benchmark of the BASELINE metric: one Gauss-Newton iteration of the
shifted-solve inversion (C4: 46^3-hex Nedelec box, N = 662,446 edge dofs,
16 poles, 4 sources x 100 receivers x 31 times, 30 LSQR iterations, RT0
regularisation lambda = 1e-2), plus its components (J v / J^T w per second,
factor FP64 TFLOP/s, solve GB/s).

A "step" is one GN iteration of `run_inversion` (inversion.py:240-300):
operator at the current model, gradient (one J^T w), LSQR (30 x (J v + J^T w)),
Armijo line search (each trial = 16 refactorisations + forward solves).

Usage (contract): python bench.py [--gpus N] [--steps K] [--warmup W]
                  [--impl ours|reference] [--config C4] [--n 46]
For N > 1 launch with torchrun; poles are sharded i -> rank (i mod N).
"""

from __future__ import annotations

import argparse
import copy
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GN-iteration s & J·v/Jᵀ·w per s at ~700k DOF; factor FP64 TFLOP/s; solve GB/s"
# line-search evaluations per GN iteration on C4 (measured by the GPU arm:
# 32 factorisations of 16 poles per GN iteration, BENCH_r01 counts)
PHI_LINE_SEARCH = 2
C1_LSQR = 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", default="C4")
    ap.add_argument("--n", type=int, default=None, help="override the mesh size (debug)")
    ap.add_argument("--lsqr", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--shard", type=int, default=0,
                    help="run only rank 0's pole shard of a G-GPU job on this GPU")
    ap.add_argument("--profile-once", action="store_true",
                    help="one factorisation + one forward only (for ncu captures)")
    ap.add_argument("--no-verify", action="store_true", help="skip the verification leg")
    ap.add_argument("--no-c1", action="store_true", help="skip the measured C1 line")
    ap.add_argument("--ref-sample", type=int, default=0,
                    help="(internal) time one C4-shape SuperLU pole at this n, print JSON")
    return ap.parse_args()


def dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # the scaling run's log shows the ranks/channels NCCL actually formed
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank


class Clocks:
    """nvidia-smi sampled during the timed region (B200_PROFILING recipe)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        dev = os.environ.get("LOCAL_RANK", "0")
        rows = [r for r in rows if r[0].strip() == dev] or rows
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            for k, name in enumerate(names):
                if len(r) > 5 + k and "Active" in r[5 + k] and "Not" not in r[5 + k]:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows)}


def measured_traffic():
    """Per-unit DRAM traffic of the factorisation / solve kernel classes from the
    committed ncu capture (profiles/dram_r01.json, tools/ncu_summary.py)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "dram_r01.json")))
    except OSError:
        return {}


def oz_roles(pr):
    """The Ozaki GEMM's own cycle counters over the timed region
    (rba_oz_prof): where its MMA-issuing thread spent its time, the SM clock it
    ran at (the INT8 phases run under the power cap) and the tensor-pipe
    occupancy they imply (28 MMAs of 128x64x32 = 896 clk per k step at peak)."""
    loop = pr.get("mma_loop", 0.0)
    if loop <= 0:
        return {}
    per_k = loop / max(pr["ksteps"], 1.0)
    return {"sm_mhz": round(1e3 * loop / max(pr["mma_loop_ns"], 1.0)),
            "clk_per_kstep": round(per_k, 1),
            "tensor_busy_frac": round(896.0 / per_k, 3),
            "wait_data_frac": round(pr["mma_wait_data"] / loop, 3),
            "wait_tmem_frac": round(pr["mma_wait_tmem"] / loop, 3),
            "ksteps_per_tile": round(pr["ksteps"] / max(pr["tiles"], 1.0), 1),
            "epilogue_clk_per_tile": round((pr["epi_drain"] + pr["epi_rmw"]) / max(pr["tiles"], 1.0))}


def measured_peaks():
    peaks = {}
    try:
        peaks.update(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))))
    except OSError:
        peaks["hbm_gbs"] = 6650.0
        peaks["_hbm_source"] = "fallback (B200_PROFILING.md)"
    try:
        fp = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")))
        peaks["fp64_tflops"] = fp["dmma_tflops"]
    except OSError:
        peaks["fp64_tflops"] = 37.0
    return peaks


def build_workload(name, n_override, lsqr_override, device=False):
    import paper_2605_19951_b200 as rb
    # device=True: topology and K generated on the GPU (mesh_gen.cu), same
    # problem as the host builder (tests/test_gpu_meshgen.py)
    prob, meta = rb.build_config(name, n=n_override, device=device)
    approx = rb.config_approximant(name)
    lsqr_iters = lsqr_override or meta.get("lsqr_iters", 30)
    return prob, meta, approx, lsqr_iters


def run_ours(args, world, rank):
    import torch
    import torch.distributed as dist
    import paper_2605_19951_b200 as rb
    from paper_2605_19951_b200.inversion import GNDriver, InversionConfig, LsqrConfig

    t_setup = time.perf_counter()
    prob, meta, approx, lsqr_iters = build_workload(args.config, args.n, args.lsqr, device=True)
    m_true = rb.Model(prob.m_true, np.full(prob.grid.cell_count, np.log(0.01)))
    cache = rb.ShiftedFactorCache()
    eps_r, seed = meta.get("noise", (0.02, 2))
    data = rb.make_dataset(prob, m_true, approx, rb.NoiseSpec(eps_r=eps_r, seed=seed), cache)
    reg = rb.build_reg(prob.grid)          # C4: face-based RT0 root (P > dense limit)
    lam = meta.get("lam", 1e-2)
    cfg = InversionConfig(lambda0=lam, lsqr=LsqrConfig(tol=0.0, max_iters=lsqr_iters),
                          m0=np.full(prob.grid.cell_count, np.log(meta.get("m0", 0.01))),
                          chi2_target=0.0)
    drv = GNDriver(prob, data, approx, cfg, cache, reg)
    eng = cache.engine
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    nu = 0
    # warm-up; the LAST warm-up step runs with per-launch CUDA events on
    # (kernel-class and per-level split); the timed region runs without them
    for k in range(args.warmup):
        if k == args.warmup - 1:
            eng.set_timing(2)
            eng.set_timing(1)
        nu += 1
        drv.iterate(nu)
    cls = eng.timings()
    lev = eng.timings_detail()
    eng.set_timing(0)
    split_fact = drv.state.history[-1].factorizations if drv.state.history else 0
    split_solves = drv.state.history[-1].solves if drv.state.history else 0
    # driver state at the start of the timed region: the e2e leg below replays
    # exactly these K GN iterations (same line-search path, same work); both
    # start with the factors and fields of the current model resident
    from paper_2605_19951_b200.forward import forward_device
    if eng.model_tag != drv.model.version_tag() or not eng.g_valid:
        forward_device(prob, drv.model, approx, cache)
    snap_keys = ("model", "g_tag", "d_pred", "misfit", "reg_val", "lam", "phi", "chi2",
                 "increase_streak")
    snap = {k: copy.deepcopy(getattr(drv, k)) for k in snap_keys}
    nu_snap = nu
    # ---- timed region: K GN iterations, inputs resident in HBM ------------
    eng.set_timing(2)                     # reset the launch counter; events stay off
    eng.oz_prof(True)                     # reset the Ozaki GEMM's role counters
    clocks = Clocks()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fac0, sol0 = cache.counters.factorizations, cache.counters.solves
    e0.record(stream)
    val_steps = []
    for _ in range(args.steps):
        nu += 1
        ts = time.perf_counter()
        drv.iterate(nu)
        val_steps.append((time.perf_counter() - ts) * 1e3)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    launches = int(eng.timings()["launches"])
    oz_prof = eng.oz_prof(True)           # cycle counters of the timed region (not a profiler)
    n_fact = cache.counters.factorizations - fac0
    n_solve = cache.counters.solves - sol0
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps

    # ---- e2e: public API with host buffers (pinned H2D of m and d_obs, D2H of
    # the updated model inside the timed region), replaying the same K GN
    # iterations from the snapshot; the factors and fields at the snapshot
    # model are restored outside the timed region ---------------------------
    for k, v in snap.items():
        setattr(drv, k, copy.deepcopy(v))
    drv.state.model, drv.state.lam = drv.model, drv.lam
    nu = nu_snap
    forward_device(prob, drv.model, approx, cache)
    m_host = torch.from_numpy(drv.model.m.copy()).pin_memory()
    d_host = torch.from_numpy(np.asarray(data.d_obs, dtype=float).copy()).pin_memory()
    out_host = torch.empty_like(m_host).pin_memory()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    clocks2 = Clocks()
    fac1, sol1 = cache.counters.factorizations, cache.counters.solves
    e2.record(stream)
    e2e_steps = []
    for _ in range(args.steps):
        nu += 1
        ts = time.perf_counter()
        m_dev = m_host.to("cuda", non_blocking=True)
        d_dev = d_host.to("cuda", non_blocking=True)
        drv.model = rb.Model(m_dev.cpu().numpy(), drv.model.m_ref)
        drv.data.d_obs = d_dev.cpu().numpy()
        drv.iterate(nu)
        out_host.copy_(torch.from_numpy(drv.model.m))
        m_host.copy_(out_host)          # the caller feeds the updated model back
        e2e_steps.append((time.perf_counter() - ts) * 1e3)
    e3.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk2 = clocks2.stop()
    e2e_detail = {"steps_wall_ms": e2e_steps, "clocks": clk2,
                  "factorizations": cache.counters.factorizations - fac1,
                  "solves": cache.counters.solves - sol1}
    e2e_ms = e2.elapsed_time(e3) / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    bytes_in = m_host.numel() * 8 + d_host.numel() * 8
    bytes_out = out_host.numel() * 8

    # ---- component rates (after the timed region) ---------------------------
    sym_flops, nnzL = symbolic_stats(eng)
    verify = verify_factors(eng, cache, prob, approx, drv.model) if not args.no_verify else None
    comp = component_rates(eng, cache, drv, sym_flops, nnzL, world)

    # ---- roofline of the dominant kernel class in the timed region ---------
    peaks = measured_peaks()
    traffic = measured_traffic()
    # kernel-class times from the instrumented last warm-up step (one GN
    # iteration: split_fact factorisations, split_solves solves)
    fact_ms = sum(cls[k] for k in ("scatter", "extend_add", "diag", "trsm", "gemm", "ozaki"))
    solve_ms = cls["solve_fwd"] + cls["solve_bwd"]
    n_local_fact = split_fact
    fact_flops = sym_flops * n_local_fact
    S = eng.S
    nr = {1: 1, 2: 2, 3: 4, 4: 4}.get(S, 8)
    solve_bytes_one = 2 * nnzL * 16 + eng.N * 16 + 4 * eng.N * nr * 16
    n_local_solve = split_solves
    if fact_ms >= solve_ms:
        achieved = fact_flops / (fact_ms * 1e-3) / 1e12
        roof = {"kernel": "frontal factorisation (K2-K4: scatter+extend-add+diag+trsm+gemm)",
                "bound": "tensor", "achieved": achieved, "peak": peaks["fp64_tflops"],
                "unit": "TFLOP/s", "frac": achieved / peaks["fp64_tflops"],
                "peak_source": "measured FP64 DMMA microbenchmark (profiles/fp64_peak_r01.json)",
                "traffic": traffic.get("factor_bytes_per_pole"),
                "traffic_unit": "DRAM bytes per pole factorisation (ncu, profiles/dram_r01.json)",
                "per_unit": "8*sum_s(p^3/6 + r p^2/2 + r^2 p/2) flops/pole",
                "note": "algorithmic (4-multiply complex) flops; the 3-multiply DMMA products "
                        "execute 3/4 of the trailing-update flops, so frac can exceed 1; "
                        "kernel times from CUDA events around every launch in the last "
                        "warm-up GN iteration (the timed region runs without events)",
                "units_per_step": n_local_fact}
    else:
        achieved = solve_bytes_one * n_local_solve / (solve_ms * 1e-3) / 1e9
        roof = {"kernel": "multifrontal triangular solves (K6/K7)", "bound": "hbm",
                "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"],
                "traffic": traffic.get("solve_bytes_per_pole_solve"),
                "traffic_unit": "DRAM bytes per pole-solve (ncu, profiles/dram_r01.json)",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "per_unit": "2*nnz(L)*16 + N*16 + 4*N*nrhs*16 bytes/solve",
                "units_per_step": n_local_solve}
    # per-kernel rooflines of the factorisation's two GEMM engines (one
    # instrumented GN iteration): the Ozaki INT8 Schur kernel against the INT8
    # dense peak (2 x the measured BF16 dense peak: same tcgen05 datapath at
    # twice the rate) and the DMMA GEMM against the measured FP64 DMMA peak
    oz = eng.oz_stats()
    rooflines = {}
    if oz["on"] and cls.get("ozaki", 0) > 0:
        try:
            pk = json.load(open(os.path.join(ROOT, "profiles", "int8_peak_r02.json")))
            # a kernel timed inside a long step: the SUSTAINED peak (same MMA loop run
            # for seconds with random operand bytes: the board power cap holds the SMs
            # at ~1.55 GHz); the burst figure is reported beside it
            int8_peak = pk.get("sustained_tops", pk["peak_tops"])
            int8_burst = pk["peak_tops"]
            int8_src = ("measured tcgen05 kind::i8 microbenchmark, sustained (power-capped) rate "
                        "(profiles/int8_peak_r02.json; burst %.0f TOPS)" % int8_burst)
        except OSError:
            int8_peak = int8_burst = 2.0 * peaks.get("bf16_tflops", 2250.0)
            int8_src = "2 x MEASURED_PEAKS.json bf16_tflops (dense INT8 = 2 x BF16 on sm_100)"
        ach = oz["int8_ops_per_pole"] * n_local_fact / (cls["ozaki"] * 1e-3) / 1e12
        rooflines["ozaki_int8_schur"] = {
            "bound": "tensor", "achieved": ach, "peak": int8_peak, "unit": "TOPS (int8)",
            "frac": ach / int8_peak, "peak_burst": int8_burst, "frac_of_burst": ach / int8_burst,
            "ms_per_step": cls["ozaki"],
            "fp64_equiv_tflops": oz["flops_per_pole"] * n_local_fact / (cls["ozaki"] * 1e-3) / 1e12,
            "peak_source": int8_src,
            "per_unit": "2*28*(128*64*32)*ksteps*tiles int8 ops per pole (7 digits, 28 pairs, "
                        "4-multiply real embedding)"}
    dmma_flops = (sym_flops - oz["flops_per_pole"] * (1 if oz["on"] else 0)
                  - getattr(symbolic_stats, "diag_trsm_flops", 0.0)) * n_local_fact
    if cls.get("gemm", 0) > 0:
        ach = dmma_flops / (cls["gemm"] * 1e-3) / 1e12
        rooflines["dmma_gemm"] = {
            "bound": "tensor", "achieved": ach, "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
            "frac": ach / peaks["fp64_tflops"], "ms_per_step": cls["gemm"],
            "peak_source": "measured FP64 DMMA microbenchmark (profiles/fp64_peak_r01.json)",
            "note": "algorithmic 4-multiply flops of the trailing / small-front Schur updates; "
                    "the 3-multiply DMMA kernel executes 3/4 of them"}
    rooflines["factorisation"] = {k: roof[k] for k in ("achieved", "unit", "peak", "frac")}
    if rooflines.get("ozaki_int8_schur") and rooflines.get("dmma_gemm"):
        dom = max(("ozaki_int8_schur", "dmma_gemm"), key=lambda k: rooflines[k]["ms_per_step"])
        try:
            oz_traffic = json.load(open(os.path.join(ROOT, "profiles", "dram_r02.json")))["ozaki_gemm_launches"]
        except (OSError, KeyError):
            oz_traffic = None
        roof = dict(rooflines[dom], kernel=dom,
                    traffic=oz_traffic if dom == "ozaki_int8_schur" else None,
                    traffic_unit="DRAM bytes of single k_oz_gemm launches (ncu --set full, profiles/dram_r02.json)",
                    units_per_step=n_local_fact)
    value = ms_step / 1e3
    line = {
        "metric": METRIC, "value": value, "unit": "s/GN-iteration", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "c128/f64", "data": "synthetic (seeded C4 stand-in, SURVEY §8d)",
        "config": {"workload": f"{args.config}: {meta['n']}^3-hex Kuhn-tet Nedelec box, "
                               f"N={eng.N} edge dofs, P={eng.P} cells, {eng.m} poles, "
                               f"{S} sources x {eng.Mr} receivers x {eng.Kt} times, "
                               f"{lsqr_iters} LSQR its, lambda={lam}",
                   "global_batch": eng.m, "parallelism": f"pole-sharded x{world}",
                   "l2": "inputs (factors, >100 GB) larger than L2; no flush needed"},
        "gpu_launches": launches,
        "components": comp,
        "kernel_ms": {k: round(v, 3) for k, v in cls.items() if k != "launches"},
        "kernel_ms_note": "one instrumented GN iteration (last warm-up step)",
        "solve_ms_by_level": {k: [x for x in v if x > 0] for k, v in lev.items()},
        "counts": {"factorizations": n_fact, "solves": n_solve},
        "roofline": roof,
        "rooflines": rooflines,
        "ozaki": dict(oz, timed_region=oz_roles(oz_prof)),
        "clocks": clk,
        "e2e": {"value": e2e_ms / 1e3, "unit": "s/GN-iteration",
                "h2d_bytes_per_step": bytes_in, "d2h_bytes_per_step": bytes_out},
        "e2e_detail": e2e_detail,
        "verify": verify,
        "steps_wall_ms": val_steps,
        "setup_s": setup_s,
        "memory_gb": {k: v / 1e9 for k, v in eng.info().items() if k.startswith("mem")},
    }
    eng.close()                          # free the C4 factors before the C1 line
    return line


def host_mass(prob, m):
    """Host restatement of assemble_M (mesh.py:348-355) for the verification
    leg: M = sum_c e^{m_c} M_c, COO -> CSR with duplicates summed."""
    import scipy.sparse as sp
    cd = prob.cell_dofs
    k = cd.shape[1]
    rows = np.repeat(cd, k, axis=1).ravel()
    cols = np.tile(cd, (1, k)).ravel()
    keep = (rows >= 0) & (cols >= 0)
    cell = np.repeat(np.arange(cd.shape[0]), k * k)[keep]
    vals = prob.mass_local.ravel()[keep] * np.exp(np.asarray(m, dtype=float))[cell]
    N = prob.K.shape[0]
    return sp.coo_matrix((vals, (rows[keep], cols[keep])), shape=(N, N)).tocsr()


def verify_factors(eng, cache, prob, approx, model, trials=3):
    """Correctness evidence for the factorisations of the benchmarked problem
    (outside the timed region): for every local pole of the factors resident
    after the timed steps, the normwise backward error |A x - b| / (|A| |x| +
    |b|) of a device solve with a random complex b (A assembled on the host,
    SciPy SpMV; the reference's residual guard is shifted.py:193-196), the
    growth max|L'|^2 / max|A| and the smallest pivot min|d| / max|A| of the
    pivot-free LDL^T; then the adjointness of J at the current model
    (sensitivity.py:175-188: reference metric and normwise)."""
    import scipy.sparse as sp
    import paper_2605_19951_b200 as rb
    t0 = time.perf_counter()
    m_fac = np.asarray(eng.last_m, dtype=float)
    M = host_mass(prob, m_fac).astype(complex)
    K = prob.K.astype(complex).tocsr()
    rng = np.random.default_rng(0)
    b = rng.standard_normal(eng.N) + 1j * rng.standard_normal(eng.N)
    rows = []
    for slot, i in enumerate(eng.local):
        xi = complex(eng.poles[i])
        A = (K - xi * M).tocsr()
        x = eng.solve(slot, b)
        nA = float(abs(A).sum(axis=1).max())
        bwd = float(np.linalg.norm(A @ x - b) / (nA * np.linalg.norm(x) + np.linalg.norm(b)))
        st = eng.factor_stats(slot)
        amax = float(abs(A).max())
        rows.append({"pole": int(i), "xi": [xi.real, xi.imag], "backward_error": bwd,
                     "growth": st["max_abs_Lp"] ** 2 / amax,
                     "min_pivot_rel": st["min_abs_sqrt_d"] ** 2 / amax,
                     "nonfinite": st["nonfinite"]})
    opr = rb.JacobianOperator(prob, model, approx, cache)
    rng = np.random.default_rng(4)
    worst = worst_n = 0.0
    for _ in range(trials):
        v = rng.standard_normal(opr.shape[1])
        w = rng.standard_normal(opr.shape[0])
        jv, jtw = opr.jvp(v), opr.vjp(w)
        lhs, rhs = float(jv @ w), float(v @ jtw)
        worst = max(worst, abs(lhs - rhs) / max(abs(lhs), abs(rhs)))
        worst_n = max(worst_n, abs(lhs - rhs) / (np.linalg.norm(jv) * np.linalg.norm(w)))
    return {"per_pole": rows,
            "max_backward_error": max(r["backward_error"] for r in rows),
            "max_growth": max(r["growth"] for r in rows),
            "min_pivot_rel": min(r["min_pivot_rel"] for r in rows),
            "adjoint_mismatch": worst, "adjoint_mismatch_normwise": worst_n,
            "adjoint_trials": trials,
            "factor_model": "the model of the factors resident after the timed steps "
                            "(sha1 " + rb.Model(m_fac, m_fac).version_tag() + ")",
            "seconds": time.perf_counter() - t0}


def symbolic_stats(eng):
    from paper_2605_19951_b200 import _lib
    from paper_2605_19951_b200._lib import ptr
    import ctypes as C
    # the engine's symbolic is internal; recompute stats through the host API on
    # the same pattern (cheap, host only)
    prob = eng.problem
    import scipy.sparse as sp
    K = sp.csr_matrix(prob.K)
    K.sort_indices()
    ip = np.ascontiguousarray(K.indptr, dtype=np.int64)
    ix = np.ascontiguousarray(K.indices, dtype=np.int32)
    co = np.ascontiguousarray(prob.dof_coords)
    h = _lib.vp()
    _lib.check(eng.lib.rba_symbolic_analyze(K.shape[0], ptr(ip), ptr(ix), ptr(co), 64,
                                            C.byref(h)))
    st = np.zeros(16, np.int64)
    ds = np.zeros(4)
    eng.lib.rba_symbolic_stats(h, ptr(st), ptr(ds))
    # diagonal-block LDL^T + TRSM flops (per 64-pivot block: 8 kb^3/6 and
    # 8 (rows below) kb^2/2): the part of the factorisation outside the GEMMs
    arrs = {}
    for name in ("npiv", "nf"):
        nb = C.c_int64()
        eng.lib.rba_symbolic_array(h, name.encode(), None, 0, C.byref(nb))
        a = np.empty(nb.value // 4, dtype=np.int32)
        eng.lib.rba_symbolic_array(h, name.encode(), ptr(a), nb.value, C.byref(nb))
        arrs[name] = a.astype(np.int64)
    eng.lib.rba_symbolic_destroy(h)
    dt = 0.0
    for p, nf in zip(arrs["npiv"], arrs["nf"]):
        for c0 in range(0, int(p), 64):
            kb = min(64, int(p) - c0)
            dt += 8.0 * kb ** 3 / 6 + 8.0 * (int(nf) - c0 - kb) * kb * kb / 2
    symbolic_stats.diag_trsm_flops = dt
    return float(ds[0]), int(st[3])


def component_rates(eng, cache, drv, flops, nnzL, world):
    import torch
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {}
    # factorisation of every local pole at the current model
    torch.cuda.synchronize()
    e0.record(stream)
    eng.factor()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    nl = len(eng.local)
    out["factor_tflops"] = flops * nl / (ms * 1e-3) / 1e12
    out["factor_ms_per_pole"] = ms / nl
    # forward solves (all local poles, S right-hand sides each)
    e0.record(stream)
    eng.forward()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    nr = {1: 1, 2: 2, 3: 4, 4: 4}.get(eng.S, 8)
    bytes_one = 2 * nnzL * 16 + eng.N * 16 + 4 * eng.N * nr * 16
    out["solve_gbs"] = bytes_one * nl / (ms * 1e-3) / 1e9
    out["solve_ms_per_pole"] = ms / nl
    v = torch.randn(eng.P, dtype=torch.float64, device="cuda")
    w = torch.randn(eng.S * eng.Kt * eng.Mr, dtype=torch.float64, device="cuda")
    # first action after the factorisation: builds the receiver Green's
    # functions Z_i = A_i^{-1} Q^T in receiver-Green mode
    info = eng.info()
    out["jvp_mode"] = "receiver-green" if info.get("green") else "sweeps"
    e0.record(stream)
    eng.jvp(v)
    e1.record(stream)
    torch.cuda.synchronize()
    out["first_jvp_ms"] = e0.elapsed_time(e1)
    reps = 3
    e0.record(stream)
    for _ in range(reps):
        eng.jvp(v)
        eng.vjp(w)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out["jv_jtw_pairs_per_s"] = 1e3 / ms
    out["factor_flops_per_pole"] = flops
    out["nnzL_per_pole"] = nnzL
    return out


def cpu_baseline_sample(name):
    """Oracle (SciPy SuperLU, the reference's backend) timed on the host on a
    bounded sample: one pole's factorisation + solves at two mesh sizes of the
    config's shape, power-law extrapolated to the config size and scaled by the
    GN-iteration count law of SURVEY §3D, pole-parallel over the host cores."""
    from oracle import rbainv_oracle as orc
    import paper_2605_19951_b200 as rb
    import scipy.sparse.linalg as spla
    cores = os.cpu_count() or 1
    spec_n = rb.config_spec(name)[1]["n"]
    approx = rb.config_approximant(name)
    pts = []
    for n in (10, 14):
        prob, _ = rb.build_config(name, n=n)
        m = prob.m_true
        t0 = time.perf_counter()
        M = orc.assemble_M(prob, m).astype(complex)
        A = (prob.K.astype(complex) - approx.poles[0] * M).tocsc()
        lu = spla.splu(A)
        tf = time.perf_counter() - t0
        rhs = prob.source_matrix().T.astype(complex)
        t0 = time.perf_counter()
        for _ in range(3):
            lu.solve(rhs)
        ts = (time.perf_counter() - t0) / 3
        pts.append((prob.dof_count, tf, ts))
    (N1, f1, s1), (N2, f2, s2) = pts
    prob_full, meta = rb.build_config(name, n=4)
    N_full = {"C1": 26416, "C4": 662446, "C5": 1798336}.get(name.upper(), N2)
    ef = math.log(f2 / f1) / math.log(N2 / N1)
    es = math.log(s2 / s1) / math.log(N2 / N1)
    tf = f2 * (N_full / N2) ** ef
    ts = s2 * (N_full / N2) ** es
    m = approx.pole_count
    itn = meta.get("lsqr_iters", 30)
    phi = PHI_LINE_SEARCH
    serial = m * phi * tf + m * (2 * itn + 2 + phi) * ts
    return {"value": serial / min(cores, m), "unit": "s/GN-iteration", "cores": min(cores, m),
            "kind": "port", "measured": False, "basis": "extrapolated",
            "sample": (f"oracle SuperLU factor+solve of 1 pole measured at N={N1} and N={N2} "
                       f"({name} shape), power-law extrapolated (factor ~N^{ef:.2f}, solve "
                       f"~N^{es:.2f}) to N={N_full}, x GN count law m*phi factorisations + "
                       f"m*(2*itn+2+phi) solves (m={m}, itn={itn}, phi={phi} = the line-search "
                       f"evaluations per GN iteration the GPU arm measures on this config), "
                       f"ideal pole-parallel on {min(cores, m)} cores; the config itself exceeds "
                       f"host RAM.  bench.py --impl reference measures the C1 GN iteration and "
                       f"C4-shape poles at n=16/20/24 (shorter reach)")}


C1_WORKLOAD = ("C1: 16^3-hex Kuhn-tet Nedelec box, N=26,416 edge dofs, P=24,576 cells, 8 poles, "
               "1 loop x 20 receivers x 31 times, 20 LSQR its, lambda=1e-2, reference dense-"
               "Cholesky R; one GN iteration of run_inversion from the homogeneous 0.01 S/m "
               "start (gradient, LSQR, Armijo line search with refactorisations)")


def c1_measured_gpu(steps=3):
    """The C1 GN iteration on the GPU through the public API, end to end:
    H2D of m and d_obs (pinned) and D2H of the updated model inside the timed
    region, CUDA events on the launching stream."""
    import torch
    import paper_2605_19951_b200 as rb
    from paper_2605_19951_b200.inversion import GNDriver, InversionConfig, LsqrConfig
    prob, meta = rb.build_config("C1")
    approx = rb.config_approximant("C1")
    m0 = np.full(prob.grid.cell_count, np.log(0.01))
    cache = rb.ShiftedFactorCache()
    data = rb.make_dataset(prob, rb.Model(prob.m_true, m0), approx,
                           rb.NoiseSpec(eps_r=0.01, seed=0), cache)
    reg = rb.build_reg(prob.grid)
    cfg = InversionConfig(lambda0=1e-2, lsqr=LsqrConfig(tol=0.0, max_iters=C1_LSQR), m0=m0,
                          chi2_target=0.0)
    drv = GNDriver(prob, data, approx, cfg, cache, reg)
    drv.iterate(1)                       # warm-up
    stream = torch.cuda.current_stream()
    m_host = torch.from_numpy(drv.model.m.copy()).pin_memory()
    d_host = torch.from_numpy(np.asarray(data.d_obs, dtype=float).copy()).pin_memory()
    out_host = torch.empty_like(m_host).pin_memory()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for k in range(steps):
        m_dev = m_host.to("cuda", non_blocking=True)
        d_dev = d_host.to("cuda", non_blocking=True)
        drv.model = rb.Model(m_dev.cpu().numpy(), drv.model.m_ref)
        drv.data.d_obs = d_dev.cpu().numpy()
        drv.iterate(2 + k)
        out_host.copy_(torch.from_numpy(drv.model.m))
        m_host.copy_(out_host)
    e1.record(stream)
    torch.cuda.synchronize()
    hist = drv.state.history[1:]
    val = e0.elapsed_time(e1) / steps / 1e3
    cache.engine.close()
    return {"value": val, "unit": "s/GN-iteration", "steps": steps, "workload": C1_WORKLOAD,
            "phi_evals": [h.phi_evals for h in hist],
            "factorizations": [h.factorizations for h in hist],
            "h2d_bytes_per_step": int(m_host.numel() * 8 + d_host.numel() * 8),
            "d2h_bytes_per_step": int(out_host.numel() * 8),
            "chi2_after": [h.chi2 for h in hist]}


def c1_measured_cpu(workers):
    """The same C1 GN iteration with the oracle (SciPy SuperLU per pole, the
    reference's backend, shifted.py:54), poles over `workers` threads as
    PoleWorkerPool (shifted.py:129-155); setup (dataset, dense-Cholesky R,
    the forward at the start model) outside the timed region, exactly as
    run_inversion computes them before its loop (inversion.py:213-235)."""
    from oracle import rbainv_oracle as orc
    import paper_2605_19951_b200 as rb
    prob, meta = rb.build_config("C1", n=int(os.environ.get("RBA_BENCH_C1_N", "16")))
    approx = rb.config_approximant("C1")
    P = prob.grid.cell_count
    m0 = np.full(P, np.log(0.01))
    fac = orc.PoleFactors(workers=workers)
    t0 = time.perf_counter()
    d_clean, _ = orc.forward_response(prob, prob.m_true, approx.poles, approx.residues, fac)
    d_obs, sigma = orc.make_dataset(d_clean, 0.01, seed=0)
    reg = orc.build_reg(prob.grid)
    W = 1.0 / sigma
    d0, g0 = orc.forward_response(prob, m0, approx.poles, approx.residues, fac)
    setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    m1, ok, eta, n_evals, _, _ = orc.gn_iteration(prob, m0, m0, approx.poles, approx.residues,
                                                  reg["R"], reg["L"], W, d_obs, 1e-2, C1_LSQR,
                                                  fac, d_pred=d0, g=g0)
    t = time.perf_counter() - t0
    return {"value": t, "unit": "s/GN-iteration", "steps": 1, "workload": C1_WORKLOAD,
            "threads": workers, "phi_evals": n_evals, "accepted": ok, "eta": eta,
            "setup_s": setup, "kind": "port (oracle restatement of the reference, SuperLU)"}


def c4_pole_sample(n):
    """One C4-shape pole with SciPy SuperLU (COLAMD, the reference's default):
    factorisation time, one 4-RHS solve time, L+U nonzeros."""
    import scipy.sparse.linalg as spla
    import paper_2605_19951_b200 as rb
    prob, _ = rb.build_config("C4", n=n)
    approx = rb.config_approximant("C4")
    M = host_mass(prob, prob.m_true).astype(complex)
    A = (prob.K.astype(complex) - approx.poles[0] * M).tocsc()
    t0 = time.perf_counter()
    lu = spla.splu(A)
    tf = time.perf_counter() - t0
    rhs = prob.source_matrix().T.astype(complex)
    t0 = time.perf_counter()
    for _ in range(2):
        lu.solve(rhs)
    ts = (time.perf_counter() - t0) / 2
    return {"n": n, "N": int(prob.dof_count), "factor_s": tf, "solve_s": ts,
            "lu_nnz": int(lu.L.nnz + lu.U.nnz)}


def workload_desc(name, n_override, lsqr_override):
    """The `config` object shared by both arms (host-only)."""
    import paper_2605_19951_b200 as rb
    prob, meta, approx, lsqr_iters = build_workload(name, n_override, lsqr_override)
    return {"workload": f"{name}: {meta['n']}^3-hex Kuhn-tet Nedelec box, "
                        f"N={prob.dof_count} edge dofs, P={prob.grid.cell_count} cells, "
                        f"{approx.pole_count} poles, {prob.source_count} sources x "
                        f"{prob.receiver_count} receivers x {approx.channels.count} times, "
                        f"{lsqr_iters} LSQR its, lambda={meta.get('lam', 1e-2)}",
            "global_batch": approx.pole_count}


def _powerlaw(Ns, ts):
    """Least-squares log-log fit t = a N^e over the samples, plus the pairwise
    exponents (their spread is the model's uncertainty)."""
    lx, ly = np.log(np.asarray(Ns, float)), np.log(np.asarray(ts, float))
    e, la = np.polyfit(lx, ly, 1)
    pair = [float((ly[k + 1] - ly[k]) / (lx[k + 1] - lx[k])) for k in range(len(lx) - 1)]
    return float(np.exp(la)), float(e), pair


def run_reference(args):
    """--impl reference: the reference's CPU path (the oracle restatement of
    the reference: SciPy SuperLU per pole, NumPy/SciPy LSQR) on the host cores.

    Measured, not modelled: the C1 GN iteration (the largest config whose
    whole GN iteration fits a CPU), with poles over min(cores, 8) threads.
    The C4 line itself cannot run on a host (one SuperLU pole at N = 662k
    needs ~125 GB), so its value is a model calibrated on three
    measured C4-shape poles at n = 16 / 20 / 24 (N = 26k / 52k / 92k, 7x reach
    instead of 38x): power-law factor / solve times x the GN count law
    m*phi factorisations + m*(2*itn+2+phi) solves, pole-parallel over as many
    cores as host RAM admits.  Everything runs once (the samples take
    minutes), concurrently: the three pole samples in single-threaded
    subprocesses, the C1 iteration in this process."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import paper_2605_19951_b200 as rb
    try:
        import psutil
        ram = int(psutil.virtual_memory().total)
        ram_avail = int(psutil.virtual_memory().available)
    except Exception:
        ram = ram_avail = 0
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    cfg = workload_desc(args.config, args.n, args.lsqr)
    ns = (16, 20, 24) if args.n is None else (max(4, args.n // 3), max(5, args.n // 2), args.n)
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1", MKL_NUM_THREADS="1")
    procs = [subprocess.Popen([sys.executable, os.path.abspath(__file__), "--ref-sample", str(n)],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, env=env)
             for n in ns]
    c1 = c1_measured_cpu(max(1, min(cores - len(ns), 8)))
    samples = []
    for pr in procs:
        out, err = pr.communicate()
        line = [ln for ln in out.splitlines() if ln.startswith("{")]
        if pr.returncode != 0 or not line:
            raise RuntimeError(f"sample failed: {err[-500:]}")
        samples.append(json.loads(line[-1]))
    Ns = [x["N"] for x in samples]
    af, ef, pf = _powerlaw(Ns, [x["factor_s"] for x in samples])
    as_, es, ps = _powerlaw(Ns, [x["solve_s"] for x in samples])
    am, em, _ = _powerlaw(Ns, [x["lu_nnz"] for x in samples])
    prob_meta = rb.config_spec(args.config, args.n)[1]
    N_full = {"C4": 662446}.get(args.config.upper(), Ns[-1]) if args.n is None else Ns[-1]
    m = rb.config_approximant(args.config).pole_count
    itn = args.lsqr or prob_meta.get("lsqr_iters", 30)
    phi = PHI_LINE_SEARCH
    tf, ts = af * N_full ** ef, as_ * N_full ** es
    mem_pole = am * N_full ** em * 16 * 1.2          # complex L+U values + index overhead
    fit = int(ram_avail // mem_pole) if ram_avail else 0
    workers = max(1, min(cores, m, fit))
    serial = m * phi * tf + m * (2 * itn + 2 + phi) * ts
    value = serial / workers

    def model_value(e_f, e_s):       # anchored at the largest measured sample
        tf_ = samples[-1]["factor_s"] * (N_full / Ns[-1]) ** e_f
        ts_ = samples[-1]["solve_s"] * (N_full / Ns[-1]) ** e_s
        return (m * phi * tf_ + m * (2 * itn + 2 + phi) * ts_) / workers
    spread = [model_value(a, b) for a, b in zip(pf, ps)]
    cb = {"value": value, "unit": "s/GN-iteration", "cores": workers, "kind": "port",
          "measured": False, "basis": "model calibrated on measured C4-shape poles",
          "host": {"cpu_count": cores, "ram_gb": ram / 1e9, "ram_available_gb": ram_avail / 1e9},
          "samples": samples,
          "factor_exponent": ef, "factor_exponent_pairwise": pf,
          "solve_exponent": es, "solve_exponent_pairwise": ps,
          "factor_s_per_pole_c4": tf,
          "value_range_pairwise_exponents": [min(spread), max(spread)] if spread else None,
          "solve_s_per_pole_c4": ts, "lu_gb_per_pole_c4": mem_pole / 1e9,
          "poles_fitting_in_ram": fit,
          "sample": (f"SciPy SuperLU (COLAMD) factor + 4-RHS solve of one C4-shape pole at "
                     f"n={ns} (N={Ns}) measured on this host, power-law fitted (factor ~N^{ef:.2f}"
                     f", solve ~N^{es:.2f}, L+U ~N^{em:.2f}) to N={N_full}; x GN count law "
                     f"m*phi factorisations + m*(2*itn+2+phi) solves (m={m}, itn={itn}, "
                     f"phi={phi}); pole-parallel over {workers} worker(s) = min(cores {cores}, "
                     f"poles {m}, poles whose ~{mem_pole / 1e9:.0f} GB factor fits in the "
                     f"{ram_avail / 1e9:.0f} GB of available RAM: {fit})"
                     + ("; NOTE: not even one C4 pole factor fits in host RAM, so the CPU "
                        "cannot run C4 at all -- the value assumes 1 worker with unlimited "
                        "memory" if fit == 0 else ""))}
    cfg["parallelism"] = (f"host: C1 measured on {c1['threads']} threads; C4 modelled on "
                          f"{workers} pole-parallel worker(s)")
    return {"impl": "reference", "metric": METRIC, "value": value,
            "unit": "s/GN-iteration", "n_gpus": 0, "steps": 1, "steps_requested": args.steps,
            "warmup": 0, "warmup_requested": args.warmup,
            "steps_note": "the reference arm measures once: its bounded samples (three SuperLU "
                          "poles up to N=92k and one C1 GN iteration) take minutes each",
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "c128/f64", "data": "synthetic", "config": cfg,
            "cpu_baseline": cb,
            "c1_measured": c1,
            "e2e": {"value": value, "unit": "s/GN-iteration", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t0}


def run_c2(args, world, rank):
    """BASELINE config 2: shifted-solve microbenchmark.  32^3-hex box, sigma
    log-uniform in [1e-3, 1] (seed 1), 16 poles; per pole factorise once, then
    solve 4 random complex RHS (unit-normal re/im).  Reports factor TFLOP/s and
    solve GB/s (algorithmic bytes 2 nnz(L) 16 + 16 N + 4 N nrhs 16)."""
    import torch
    import paper_2605_19951_b200 as rb
    from paper_2605_19951_b200.engine import Engine
    prob, meta, approx, _ = build_workload("C2", args.n, None)
    rng = np.random.default_rng(1)
    F = rng.standard_normal((4, prob.dof_count)) + 1j * rng.standard_normal((4, prob.dof_count))
    eng = Engine(prob, None)
    eng.set_sources(F)
    eng.set_poles(approx)
    eng.set_model(prob.m_true)
    flops, nnzL = symbolic_stats(eng)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(args.warmup):
        eng.factor()
        eng.forward()
    tf, ts = [], []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        e0.record(stream)
        eng.factor()
        e1.record(stream)
        torch.cuda.synchronize()
        tf.append(e0.elapsed_time(e1))
        e0.record(stream)
        eng.forward()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    nl = len(eng.local)
    bytes_one = 2 * nnzL * 16 + eng.N * 16 + 4 * eng.N * 4 * 16
    fac_tf = flops * nl / (np.mean(tf) * 1e-3) / 1e12
    sol_gbs = bytes_one * nl / (np.mean(ts) * 1e-3) / 1e9
    peaks = measured_peaks()
    return {"metric": METRIC, "value": fac_tf, "unit": "factor FP64 TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128/f64",
            "data": "synthetic (seed 1)",
            "config": {"workload": f"C2: {meta['n']}^3 hexes, N={eng.N}, {eng.m} poles, "
                                   f"4 random complex RHS"},
            "solve_gbs": sol_gbs, "factor_ms_per_pole": float(np.mean(tf)) / nl,
            "solve_ms_per_pole": float(np.mean(ts)) / nl,
            "roofline": {"factor": {"achieved": fac_tf, "peak": peaks["fp64_tflops"],
                                    "unit": "TFLOP/s", "frac": fac_tf / peaks["fp64_tflops"]},
                         "solve": {"achieved": sol_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                   "frac": sol_gbs / peaks["hbm_gbs"]}},
            "flops_per_pole": flops, "nnzL_per_pole": nnzL}


def run_c3(args, world, rank):
    """BASELINE config 3: Jacobian operator benchmark on the 32^3 box (two 6^3
    blocks, 4 loop sources, 10x10 receivers, 31 times, 16 poles): 50 J v and
    50 J^T w with the adjointness check <Jv, w> = <v, J^T w>."""
    import torch
    import paper_2605_19951_b200 as rb
    prob, meta, approx, _ = build_workload("C3", args.n, None)
    model = prob.true_model()
    cache = rb.ShiftedFactorCache()
    opr = rb.JacobianOperator(prob, model, approx, cache)
    eng = opr.engine
    rng = np.random.default_rng(3)
    trials = 50 if args.steps >= 2 else 5
    V = torch.as_tensor(rng.standard_normal((trials, opr.shape[1])), device="cuda")
    Wt = torch.as_tensor(rng.standard_normal((trials, opr.shape[0])), device="cuda")
    for _ in range(args.warmup):
        opr.jvp_d(V[0])
        opr.vjp_d(Wt[0])
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    jv = [opr.jvp_d(V[k]) for k in range(trials)]
    jt = [opr.vjp_d(Wt[k]) for k in range(trials)]
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    worst = 0.0
    worst_n = 0.0
    for k in range(trials):
        lhs = float(torch.dot(jv[k], Wt[k]))
        rhs = float(torch.dot(V[k], jt[k]))
        worst = max(worst, abs(lhs - rhs) / max(abs(lhs), abs(rhs)))
        scale = float(torch.linalg.vector_norm(jv[k]) * torch.linalg.vector_norm(Wt[k]))
        worst_n = max(worst_n, abs(lhs - rhs) / scale)
    return {"metric": METRIC, "value": 2 * trials / (ms * 1e-3), "unit": "J·v or Jᵀ·w per s",
            "n_gpus": world, "steps": trials, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128/f64",
            "data": "synthetic (seed 3)",
            "config": {"workload": f"C3: {meta['n']}^3 hexes, N={eng.N}, P={eng.P}, {eng.m} "
                                   f"poles, {eng.S} sources x {eng.Mr} receivers x {eng.Kt} times"},
            "adjoint_max_mismatch": worst,
            "adjoint_max_mismatch_normwise": worst_n,
            "adjoint_note": "reference metric |<Jv,w>-<v,J^T w>|/max(|.|) (sensitivity.py:"
                            "175-188) is inflated when a random pair nearly cancels; the "
                            "normwise |.|/(|Jv||w|) is scale-free",
            "ms_per_action": ms / (2 * trials)}


def run_shard(args, world, rank):
    """Per-rank workload of a G-GPU run on ONE GPU: the poles rank 0 owns
    (i mod G == 0), factorised and solved (forward, J v and J^T w partials,
    without the cross-rank exchange).  Used for C5 (20 poles, 8 sources,
    n = 64: 33 GB of factor per pole), which only fits when sharded."""
    import torch
    import paper_2605_19951_b200 as rb
    from paper_2605_19951_b200.engine import Engine
    from paper_2605_19951_b200.parallel import ShardComm
    from paper_2605_19951_b200 import _lib
    from paper_2605_19951_b200._lib import ptr
    G = args.shard
    prob, meta, approx, lsqr_iters = build_workload(args.config, args.n, args.lsqr, device=True)
    eng = Engine(prob, approx, comm=ShardComm(G, 0))   # rank 0's poles, no collective
    eng.set_model(prob.m_true)
    flops, nnzL = symbolic_stats(eng)
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    v = torch.randn(eng.P, dtype=torch.float64, device="cuda")
    w = torch.randn(eng.S * eng.Kt * eng.Mr, dtype=torch.float64, device="cuda")
    for _ in range(max(1, args.warmup)):
        eng.factor()
        _lib.check(eng.lib.rba_forward_partial(eng.ctx, ptr(eng.qpart)))
    torch.cuda.synchronize()
    # first action after the factorisation builds the receiver Green's
    # functions (Green mode); timed separately, counted once per GN iteration
    t0 = time.perf_counter()
    _lib.check(eng.lib.rba_jvp_partial(eng.ctx, ptr(v), ptr(eng.qpart)))
    torch.cuda.synchronize()
    t_first = (time.perf_counter() - t0) * 1e3
    walls = []
    for step in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if step == 0:
            eng.factor()
        elif step == 1:
            eng.set_timing(2)
            eng.set_timing(1)
            _lib.check(eng.lib.rba_forward_partial(eng.ctx, ptr(eng.qpart)))
            torch.cuda.synchronize()
            fwd_levels = eng.timings_detail()
            eng.set_timing(0)
        elif step == 2:
            _lib.check(eng.lib.rba_jvp_partial(eng.ctx, ptr(v), ptr(eng.qpart)))
        else:
            _lib.check(eng.lib.rba_vjp_partial(eng.ctx, ptr(w), ptr(eng.tpart)))
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t0) * 1e3)
        if step == 1:
            # rebuild Z for the refactorised poles outside the timed actions
            t1 = time.perf_counter()
            _lib.check(eng.lib.rba_jvp_partial(eng.ctx, ptr(v), ptr(eng.qpart)))
            torch.cuda.synchronize()
            t_first = (time.perf_counter() - t1) * 1e3
    tf, tfw, tj, tv = walls
    nl = len(eng.local)
    nr = {1: 1, 2: 2, 3: 4, 4: 4}.get(eng.S, 8)
    bytes_one = 2 * nnzL * 16 + eng.N * 16 + 4 * eng.N * nr * 16
    phi = 2
    green = bool(eng.info().get("green"))
    zb = max(0.0, t_first - tj) if green else 0.0     # Z build (first action minus a steady J v)
    proj = phi * (tf + tfw) + zb + (2 * lsqr_iters + 2) * 0.5 * (tj + tv)
    peaks = measured_peaks()
    fac_tf = flops * nl / (tf * 1e-3) / 1e12
    return {"metric": METRIC, "value": proj / 1e3,
            "unit": "s/GN-iteration (projected per-rank, no exchange)", "n_gpus": 1,
            "shard_of": G, "steps": 1, "warmup": args.warmup, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128/f64", "data": "synthetic",
            "config": {"workload": f"{args.config} rank-0 shard of {G}: {meta['n']}^3 hexes, "
                                   f"N={eng.N}, poles {eng.local} of {eng.m}, {eng.S} sources x "
                                   f"{eng.Mr} receivers x {eng.Kt} times"},
            "factor_ms": tf, "forward_ms": tfw, "jvp_ms": tj, "vjp_ms": tv,
            "jvp_mode": "receiver-green" if green else "sweeps", "green_build_ms": zb,
            "forward_ms_by_level": {k: [round(x, 2) for x in v if x > 0]
                                    for k, v in fwd_levels.items() if k.startswith("solve")},
            "factor_tflops": fac_tf, "solve_gbs": bytes_one * nl / (tfw * 1e-3) / 1e9,
            "roofline": {"bound": "tensor", "achieved": fac_tf, "peak": peaks["fp64_tflops"],
                         "unit": "TFLOP/s", "frac": fac_tf / peaks["fp64_tflops"],
                         "note": "algorithmic 4-multiply flops; 3-multiply DMMA products "
                                 "execute 3/4 of them, so frac can exceed 1"},
            "flops_per_pole": flops, "nnzL_per_pole": nnzL,
            "memory_gb": {k: v / 1e9 for k, v in eng.info().items() if k.startswith("mem")},
            "note": "projection = 2 line-search evals x (factor + forward) + one Z build "
                    "(Green mode) + (2*itn+2) x mean(J v, J^T w) partial times; the all-gather "
                    "(<0.1 ms over NVLink for these sizes) is not included"}


def main():
    args = parse()
    if args.ref_sample:
        print(json.dumps(c4_pole_sample(args.ref_sample)))
        return
    if args.impl == "reference":
        line = run_reference(args)
        if line is not None:
            print(json.dumps(line))
        return
    world, rank = dist_setup(args)
    if args.shard > 1:
        line = run_shard(args, world, rank)
        print(json.dumps(line))
        return
    if args.config.upper() in ("C2", "C3"):
        line = (run_c2 if args.config.upper() == "C2" else run_c3)(args, world, rank)
        if rank == 0:
            print(json.dumps(line))
        return
    line = run_ours(args, world, rank)
    if world == 1 and not args.no_c1 and args.config.upper() == "C4":
        import torch
        torch.cuda.empty_cache()
        try:
            line["c1_measured"] = c1_measured_gpu()
        except Exception as exc:
            line["c1_measured"] = {"error": repr(exc)}
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline_sample(args.config)
        except Exception as exc:       # keep the GPU line even if the sample fails
            line["cpu_baseline"] = {"error": repr(exc)}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
