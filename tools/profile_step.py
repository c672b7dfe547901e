"""One factorisation of every pole + one forward, J v and J^T w at a BASELINE
config -- the short command used for ncu captures (no timing loop)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--n", type=int, default=None)
    args = ap.parse_args()
    import torch
    import paper_2605_19951_b200 as rb
    torch.cuda.set_device(0)
    prob, meta = rb.build_config(args.config, n=args.n)
    approx = rb.config_approximant(args.config)
    m = np.full(prob.grid.cell_count, np.log(0.01))
    model = rb.Model(m, m)
    cache = rb.ShiftedFactorCache()
    d = rb.forward_response(prob, model, approx, cache).data
    opr = rb.JacobianOperator(prob, model, approx, cache)
    jv = opr.jvp(np.ones(opr.shape[1]))
    jt = opr.vjp(np.ones(opr.shape[0]))
    torch.cuda.synchronize()
    print("ok", d.size, float(np.linalg.norm(jv)), float(np.linalg.norm(jt)))


if __name__ == "__main__":
    main()
