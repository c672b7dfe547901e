"""C4 receiver-Green build (Z_i = A_i^-1 Q^T): time of the first J v after a
factorisation (the build) and of the streamed actions; prints a checksum of
J v so variants (env) can be compared.  python tools/green_check.py"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19951_b200 as rb

prob, _ = rb.build_config(os.environ.get("CFG", "C4"))
approx = rb.config_approximant(os.environ.get("CFG", "C4"))
model = rb.Model(prob.m_true, prob.m_true)
cache = rb.ShiftedFactorCache()
rb.forward_response(prob, model, approx, cache)
opr = rb.JacobianOperator(prob, model, approx, cache)
eng = cache.engine
rng = np.random.default_rng(0)
v = rng.standard_normal(opr.shape[1]); w = rng.standard_normal(opr.shape[0])
def timed(f):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); out = f(); e1.record(); torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)
eng.set_timing(2); eng.set_timing(1)
jv, t_first = timed(lambda: opr.jvp(v))
cls = eng.timings(); eng.set_timing(0)
jv2, t_jv = timed(lambda: opr.jvp(v))
jtw, t_jtw = timed(lambda: opr.vjp(w))
print(f"first J v (Z build + action) {t_first:.1f} ms; classes green {cls['green']:.1f} solve_fwd {cls['solve_fwd']:.1f}; "
      f"J v {t_jv:.2f} ms, J^T w {t_jtw:.2f} ms")
print("adjoint mismatch", abs(np.vdot(jv, w) - np.vdot(v, jtw)) / abs(np.vdot(jv, w)))
np.save(os.environ.get("OUT", "/tmp/jv.npy"), np.concatenate([jv, jtw]))
