"""C4 multi-RHS solves only: one factorisation, then forward() sweeps (16 poles,
4 right-hand sides) timed with CUDA events and split per level.
python tools/solve_check.py [n_forward]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19951_b200 as rb
from paper_2605_19951_b200.engine import Engine

nrep = int(sys.argv[1]) if len(sys.argv) > 1 else 3
prob, _ = rb.build_config(os.environ.get("CFG", "C4"))
approx = rb.config_approximant(os.environ.get("CFG", "C4"))
eng = Engine(prob, approx)
eng.set_model(prob.m_true)
eng.factor()
torch.cuda.synchronize()
ts = []
for _ in range(nrep):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); eng.forward(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
info = eng.info()
nnz = float(os.environ.get("NNZL", 458722054))
m = len(approx.poles)
alg = m * (2 * nnz * 16 + eng.N * 16 + 4 * eng.N * 4 * 16)
print(f"forward() {min(ts):.2f} ms (all {[round(t, 2) for t in ts]}): {alg / min(ts) / 1e6:.0f} GB/s algorithmic")
if nrep > 1:
    eng.set_timing(2); eng.set_timing(1); eng.forward(); lev = eng.timings_detail(); cls = eng.timings(); eng.set_timing(0)
    print(f"fwd {cls['solve_fwd']:.2f} bwd {cls['solve_bwd']:.2f} elem {cls['elem']:.2f}")
    print("solve_fwd_by_level", [round(x, 2) for x in lev["solve_fwd_by_level"][:15]])
    print("solve_bwd_by_level", [round(x, 2) for x in lev["solve_bwd_by_level"][:15]])
