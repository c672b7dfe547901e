"""C4 factorisation time and per-pole backward error, DMMA vs Ozaki (INT8)
Schur updates: python tools/oz_check.py  (env RBA_OZAKI selects the path)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19951_b200 as rb
from paper_2605_19951_b200.engine import Engine
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

prob, _ = rb.build_config("C4")
approx = rb.config_approximant("C4")
eng = Engine(prob, approx)
eng.set_model(prob.m_true)
eng.factor()
torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); eng.factor(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
eng.set_timing(2); eng.set_timing(1); eng.factor(); cls = eng.timings(); lev = eng.timings_detail(); eng.set_timing(0)
eng.oz_prof(True); eng.factor(); pr = eng.oz_prof(True)
if pr["mma_loop"] > 0:
    print("oz_prof (fractions of the MMA-issuer loop):",
          {k: round(v / pr["mma_loop"], 3) for k, v in pr.items() if k not in ("ksteps", "tiles", "mma_loop_ns")},
          "SM MHz", round(1e3 * pr["mma_loop"] / max(pr["mma_loop_ns"], 1)),
          "clk per k step", round(pr["mma_loop"] / max(pr["ksteps"], 1), 1),
          "k steps per tile", round(pr["ksteps"] / max(pr["tiles"], 1), 1),
          "clk per tile: drain", round(pr["epi_drain"] / max(pr["tiles"], 1)),
          "rmw", round(pr["epi_rmw"] / max(pr["tiles"], 1)),
          "GEMM busy ms (issuer loops / 148 SMs)", round(pr["mma_loop_ns"] / 148e6, 1))
print("factor_by_level", [round(x, 1) for x in lev["factor_by_level"][:15]])
print("gemm_by_level", [round(x, 1) for x in lev["gemm_by_level"][:15]])
print("classes", {k: round(v, 1) for k, v in cls.items()})
M = bench.host_mass(prob, prob.m_true).astype(complex)
K = prob.K.astype(complex).tocsr()
rng = np.random.default_rng(0)
b = rng.standard_normal(eng.N) + 1j * rng.standard_normal(eng.N)
out = []
for i in (0, 8, 15):
    A = (K - approx.poles[i] * M).tocsr()
    x = eng.solve(i, b)
    nA = abs(A).sum(axis=1).max()
    out.append(float(np.linalg.norm(A @ x - b) / (nA * np.linalg.norm(x) + np.linalg.norm(b))))
print(f"RBA_OZAKI={os.environ.get('RBA_OZAKI','0')}: factor 16 poles {min(ts):.1f} ms "
      f"gemm {cls['gemm']:.1f} ms; backward {out}; mem {eng.info()['mem_work']/1e9:.1f} GB work", flush=True)
# forward solves of all 16 poles (4 RHS): per-level split of one instrumented call
eng.forward(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); eng.forward(); e1.record(); torch.cuda.synchronize()
tsol = e0.elapsed_time(e1)
eng.set_timing(2); eng.set_timing(1); eng.forward(); lev = eng.timings_detail(); cls = eng.timings(); eng.set_timing(0)
print(f"forward (16 poles, 4 RHS): {tsol:.2f} ms; fwd {cls['solve_fwd']:.2f} bwd {cls['solve_bwd']:.2f} elem {cls['elem']:.2f}")
print("solve_fwd_by_level", [round(x, 2) for x in lev["solve_fwd_by_level"][:15]])
print("solve_bwd_by_level", [round(x, 2) for x in lev["solve_bwd_by_level"][:15]])
