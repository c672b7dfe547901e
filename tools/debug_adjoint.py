"""Adjointness of the device J / J^T at the C3 shape for several mesh sizes and
models (random v, w as in the reference's adjoint_test)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_19951_b200 as rb
torch.cuda.set_device(0)
for n in [int(a) for a in sys.argv[1:]]:
    prob, _ = rb.build_config("C3", n=n)
    ap = rb.config_approximant("C3")
    for label, m in (("true(air)", prob.m_true), ("no-air", np.where(prob.m_true < np.log(1e-6), np.log(0.01), prob.m_true))):
        model = rb.Model(m, m)
        cache = rb.ShiftedFactorCache()
        opr = rb.JacobianOperator(prob, model, ap, cache)
        rng = np.random.default_rng(3)
        worst = 0
        for k in range(5):
            v = rng.standard_normal(opr.shape[1]); w = rng.standard_normal(opr.shape[0])
            l = opr.jvp(v) @ w; r = v @ opr.vjp(w)
            worst = max(worst, abs(l - r) / max(abs(l), abs(r)))
            if k == 0: print(n, label, l, r)
        d = rb.forward_response(prob, model, ap, cache).data
        np.save(f"gpurun_out/c3_gpu_d_n{n}_{label[:4]}.npy", d)
        print(f"C3 n={n} {label}: adjoint worst {worst:.3e}", flush=True)
        cache.engine.close()
