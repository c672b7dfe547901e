"""Check the per-rank shard path: forward partial timing and values vs single-pole solves."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_19951_b200 as rb
from paper_2605_19951_b200.engine import Engine
from paper_2605_19951_b200.parallel import PoleComm
from paper_2605_19951_b200 import _lib
from paper_2605_19951_b200._lib import ptr
torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
prob, meta = rb.build_config("C5", n=n)
approx = rb.config_approximant("C5")
eng = Engine(prob, approx, comm=PoleComm(8, 0))
eng.set_model(prob.m_true)
eng.set_timing(1)
eng.factor(); torch.cuda.synchronize()
t = time.perf_counter()
_lib.check(eng.lib.rba_forward_partial(eng.ctx, ptr(eng.qpart))); torch.cuda.synchronize()
print("forward_partial wall ms", (time.perf_counter() - t) * 1e3, eng.timings())
g = eng.download_g(0)
F = prob.source_matrix()
x = eng.solve(0, F[0].astype(complex))
print("g vs solve rel", np.linalg.norm(g[:, 0] - x) / np.linalg.norm(x))
