"""Generate the committed golden vectors from the UNMODIFIED reference.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py [--c1]

Outputs (small .npz / .json files next to this script, plus the frozen
approximants under paper_2605_19951_b200/data/):

* ``approx_C{1,2,3,4,5}.json`` -- `rbainv.fit_common_pole` approximants for the
  BASELINE configs (rba.py:280-378), each fitted on its own config's spectral
  interval, saved with `rbainv.save_approximant`.
* ``ref2d_small.npz``   -- the reference's own 2-D `small_problem` fixture
  (pkg/tests/conftest.py:28-47) with its arrays and the reference outputs:
  pole solutions, forward data, J v, J^T w, adjoint mismatch, LSQR updates.
* ``ref3d_n6.npz`` / ``ref3d_c3_n6.npz`` -- 3-D Nedelec problems built by
  paper_2605_19951_b200.mesh3d fed through the reference's own functions
  (single source, and a 4-source problem composed per source).
* ``ref3d_C1.npz`` (--c1) -- the C1 configuration at full size (n=16) at the
  homogeneous start model.
* ``ref3d_C1_true.npz`` (--c1true) -- C1 at full size at its TRUE model
  (1e-8 S/m air, 1 S/m block, 0.01 S/m half-space), m_ref = start model:
  forward data, J v, J^T w, adjointness, the GN update after 1/3/5/20 LSQR
  iterations with the reference's dense-Cholesky R, the reference's own
  solver-to-solver floor on those updates (SuperLU COLAMD vs MMD_AT_PLUS_A,
  oracle/rbainv_oracle.lsqr_floor, itself pinned to the reference), the
  robust secondaries after the step (phi, chi^2, linearised residual), and
  checks of the reference R (R u, R^T y, nnz, sha256).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import rbainv as rb  # noqa: E402  (the reference)

from paper_2605_19951_b200 import mesh3d  # noqa: E402

DATA = os.path.join(REPO, "paper_2605_19951_b200", "data")


def fit_approximants():
    os.makedirs(DATA, exist_ok=True)
    out = {}
    for name, n_poles, (t0, t1, nt) in (("C1", 8, (1e-5, 1e-2, 31)),
                                        ("C2", 16, (1e-5, 1e-2, 31)),
                                        ("C3", 16, (1e-5, 1e-2, 31)),
                                        ("C4", 16, (1e-5, 1e-2, 31)),
                                        ("C5", 20, (1e-6, 1e-2, 41))):
        path = os.path.join(DATA, f"approx_{name}.json")
        if os.path.exists(path):
            out[name] = rb.load_approximant(path)
            continue
        # spectral interval: element-pencil bound of the config's true model
        # (air at 1e-8 S/m dominates), 5% margin -- as rba fixtures do.
        if name in ("C3", "C4"):
            # each config on its own interval: the full-size true model's
            # element-pencil bound (its 1e-8 S/m air dominates)
            prob, _ = mesh3d.build_config(name)
        else:
            prob, _ = mesh3d.build_config("C2" if name == "C2" else "C1", n=8)
        bound = mesh3d.spectral_bound(prob, prob.m_true)
        if name == "C2":
            bound = mesh3d.spectral_bound(prob, np.full(prob.grid.cell_count, np.log(1e-3)))
        t = time.time()
        ap = rb.fit_common_pole(rb.TimeChannels.logspaced(t0, t1, nt), (0.0, 1.05 * bound),
                                n_poles)
        print(f"fit {name}: {n_poles} poles, err {ap.fit_error:.3e}, converged {ap.converged},"
              f" {time.time() - t:.1f}s, Re>0: {(ap.poles.real > 0).sum()}")
        rb.save_approximant(ap, path)
        out[name] = ap
    return out


def receiver_grid(lo, hi, n):
    xs = np.linspace(lo, hi, n)
    return np.array([(x, y) for y in xs for x in xs])


def ref_outputs(problem, model, approx, reg, data, seeds=(3, 4), lsqr_iters=(1, 3, 5),
                lam=1e-2, sources=None):
    """Run the reference's own path; sources (S,N) composes per-source."""
    F = [problem.f] if sources is None else list(sources)
    Kt, Mr = approx.channels.count, problem.Q.shape[0]
    P = model.cell_count
    out = {}
    caches, oprs, datas, gs = [], [], [], []
    for s, f in enumerate(F):
        problem.f = np.asarray(f, dtype=float)
        cache = rb.ShiftedFactorCache()
        g = rb.solve_all_poles(problem, model, approx, problem.f, cache)
        d, _ = rb.response_from_pole_solutions(problem, approx, g)
        opr = rb.JacobianOperator(problem, model, approx, cache, pole_solutions=g)
        caches.append(cache)
        oprs.append(opr)
        datas.append(d)
        gs.append(g)
    problem.f = np.asarray(F[0], dtype=float)
    out["g"] = np.stack(gs, axis=2)                     # (m, N, S)
    out["d"] = np.concatenate(datas)
    rng = np.random.default_rng(seeds[0])
    v = rng.standard_normal(P)
    w = rng.standard_normal(len(F) * Kt * Mr)
    out["v"], out["w"] = v, w
    out["jv"] = np.concatenate([o.jvp(v) for o in oprs])
    ws = w.reshape(len(F), Kt * Mr)
    jtw = None
    for s, o in enumerate(oprs):
        part = o.vjp(ws[s])
        jtw = part if jtw is None else jtw + part
    out["jtw"] = jtw

    class Stacked:
        shape = (len(F) * Kt * Mr, P)

        def jvp(self, x):
            return np.concatenate([o.jvp(x) for o in oprs])

        def vjp(self, y):
            ys = np.asarray(y).reshape(len(F), Kt * Mr)
            acc = None
            for s2, o in enumerate(oprs):
                part = o.vjp(ys[s2])
                acc = part if acc is None else acc + part
            return acc

    st = Stacked()
    out["adjoint"] = np.array(rb.adjoint_test(st, trials=3, seed=seeds[1]))
    if data is not None and reg is not None:
        out["d_obs"], out["sigma_d"] = data.d_obs, data.sigma_d
        out["lam"] = np.array(lam)
        for k in lsqr_iters:
            dm, itn, istop = rb.inversion._augmented_lsqr(
                st, reg, data, out["d"], model, lam, rb.LsqrConfig(tol=0.0, max_iters=k))
            out[f"dm_{k}"] = dm
            out[f"itn_{k}"] = np.array(itn)
    return out


def save_problem_arrays(prefix, problem):
    K = problem.K.tocsr()
    Q = problem.Q.tocsr()
    g = problem.grid
    return {
        f"{prefix}K_data": K.data, f"{prefix}K_indices": K.indices, f"{prefix}K_indptr": K.indptr,
        f"{prefix}Q_data": Q.data, f"{prefix}Q_indices": Q.indices, f"{prefix}Q_indptr": Q.indptr,
        f"{prefix}Q_shape": np.array(Q.shape),
        f"{prefix}cell_dofs": problem.cell_dofs, f"{prefix}mass_local": problem.mass_local,
        f"{prefix}f": problem.f, f"{prefix}cell_measure": g.cell_measure,
        f"{prefix}face_cells": g.face_cells, f"{prefix}face_measure": g.face_measure,
    }


def approx_arrays(ap):
    return {"poles": ap.poles, "residues": ap.residues, "times": ap.channels.times}


def golden_2d():
    spec = rb.ProblemSpec(
        dimension=2, extent=(-60.0, 60.0, -60.0, 60.0), n_cells=(8, 8), kappa=1e5,
        sigma_background=0.1, receivers=receiver_grid(-45.0, 45.0, 3),
        source=rb.SourceSpec(kind="box", center=(0.0, 0.0), size=(40.0, 40.0)),
        anomalies=(rb.AnomalySpec(box=(-40, -10, -40, -10), sigma=1.0, name="cond"),))
    prob = rb.build_problem(spec)
    channels = rb.TimeChannels.logspaced(1e-6, 1e-3, 7)
    bound = rb.spectral_bound(prob, prob.reference_model())
    ap = rb.fit_common_pole(channels, (0.0, 30.0 * bound), 16, rb.FitConfig(n_log=500, n_lin=500))
    model = prob.true_model()
    reg = rb.build_reg(prob.grid)
    data = rb.make_dataset(prob, model, ap, rb.NoiseSpec(eps_r=0.02, seed=0))
    start = prob.reference_model()
    outs = ref_outputs(prob, start, ap, reg, data, lsqr_iters=(1, 3, 5, 20))
    outs.update(save_problem_arrays("", prob))
    outs.update(approx_arrays(ap))
    outs["m"] = start.m
    outs["m_ref"] = start.m_ref
    outs["m_true"] = model.m
    outs["R_dense"] = reg.R_factor.toarray()
    np.savez_compressed(os.path.join(HERE, "ref2d_small.npz"), **outs)
    print("ref2d_small: N", prob.dof_count, "P", prob.grid.cell_count)


def golden_3d(name, n, approx, fname, lsqr_iters=(1, 3, 5), dense_reg=True):
    prob, meta = mesh3d.build_config(name, n=n)
    prob.ensure_scatter()
    m_start = np.full(prob.grid.cell_count, np.log(prob.sigma_background))
    model_true = rb.Model(prob.m_true, m_start)
    model = rb.Model(m_start, m_start)
    t = time.time()
    reg = rb.build_reg(prob.grid) if dense_reg else None
    src = prob.sources if prob.sources.shape[0] > 1 else None
    # synthetic data: reference make_dataset per source, noise over the stack
    d_true = []
    for f in prob.source_matrix():
        prob.f = f
        d_true.append(rb.forward_response(prob, model_true, approx, rb.ShiftedFactorCache()).data)
    prob.f = prob.source_matrix()[0]
    d_clean = np.concatenate(d_true)
    eps_r, seed = meta.get("noise", (0.01, 0))
    eps_a = 1e-6 * np.max(np.abs(d_clean))
    sigma = np.abs(d_clean) * eps_r + eps_a
    rng = np.random.default_rng(seed)
    d_obs = d_clean + sigma * rng.standard_normal(d_clean.size)
    data = rb.DataSet(d_obs=d_obs, sigma_d=sigma, times=approx.channels.times,
                      receivers=prob.receivers, eps_r=eps_r, eps_a=eps_a, seed=seed,
                      provenance={})
    outs = ref_outputs(prob, model, approx, reg, data, lsqr_iters=lsqr_iters, sources=src)
    if prob.source_count > 1:
        outs.pop("g")
    outs["d_clean"] = d_clean
    outs["m"] = m_start
    outs["n"] = np.array(n)
    outs["name"] = np.array(name)
    if n <= 6:
        outs.update(save_problem_arrays("", prob))
    np.savez_compressed(os.path.join(HERE, fname), **outs)
    print(f"{fname}: N {prob.dof_count} P {prob.grid.cell_count} S {prob.source_count}"
          f" adjoint {float(outs['adjoint']):.2e} {time.time() - t:.1f}s")


def golden_c1_true(approx, fname="ref3d_C1_true.npz", n=16, lam=1e-2, iters=(1, 3, 5, 20)):
    import hashlib
    import scipy.sparse.linalg as spla
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import rbainv_oracle as orc          # the floor only (pinned to the reference)
    t = time.time()
    prob, meta = mesh3d.build_config("C1", n=n)
    prob.ensure_scatter()
    P = prob.grid.cell_count
    m_ref = np.full(P, np.log(prob.sigma_background))
    model = rb.Model(prob.m_true, m_ref)
    reg = rb.build_reg(prob.grid)
    print(f"build_reg {time.time() - t:.1f}s", flush=True)
    cache = rb.ShiftedFactorCache()
    eps_r, seed = meta["noise"]
    data = rb.make_dataset(prob, model, approx, rb.NoiseSpec(eps_r=eps_r, seed=seed), cache)
    g = rb.solve_all_poles(prob, model, approx, prob.f, cache)
    d, _ = rb.response_from_pole_solutions(prob, approx, g)
    opr = rb.JacobianOperator(prob, model, approx, cache, pole_solutions=g)
    out = {"m": prob.m_true, "m_ref": m_ref, "n": np.array(n), "lam": np.array(lam),
           "d": d, "d_obs": data.d_obs, "sigma_d": data.sigma_d}
    rng = np.random.default_rng(3)
    v = rng.standard_normal(P)
    w = rng.standard_normal(d.size)
    out.update(v=v, w=w, jv=opr.jvp(v), jtw=opr.vjp(w))
    out["adjoint"] = np.array(rb.adjoint_test(opr, trials=3, seed=4))
    print(f"forward/J done {time.time() - t:.1f}s", flush=True)
    W = data.weights
    sql = np.sqrt(lam)
    R = reg.R_factor
    for k in iters:
        dm, itn, istop = rb.inversion._augmented_lsqr(opr, reg, data, d, model, lam,
                                                      rb.LsqrConfig(tol=0.0, max_iters=k))
        out[f"dm_{k}"], out[f"itn_{k}"] = dm, np.array(itn)
        # linearised residual of the augmented system after the step
        r1 = W * (opr.jvp(dm) + d - data.d_obs)
        r2 = sql * (R @ (dm + model.m - m_ref))
        out[f"linres_{k}"] = np.array(np.sqrt(r1 @ r1 + r2 @ r2))
        if k in (5, 20):
            trial = rb.Model(model.m + dm, m_ref)
            dn = rb.forward_response(prob, trial, approx, rb.ShiftedFactorCache()).data
            mis = 0.5 * float(np.sum((W * (dn - data.d_obs)) ** 2))
            rv, _ = rb.reg_value_grad(reg, trial)
            out[f"phi_{k}"] = np.array(mis + lam * rv)
            out[f"chi2_{k}"] = np.array(2.0 * mis / d.size)
            floor, dms = orc.lsqr_floor(prob, model.m, approx.poles, approx.residues, R, W,
                                        data.d_obs, lam, k, m_ref=m_ref, return_all=True)
            out[f"floor_{k}"] = np.array(floor)
            # the same secondaries for both orderings' updates: their spread is
            # the reference's own floor on phi / chi^2 / linearised residual
            sec = []
            for dmo in dms:
                r1o = W * (opr.jvp(dmo) + d - data.d_obs)
                r2o = sql * (R @ (dmo + model.m - m_ref))
                tro = rb.Model(model.m + dmo, m_ref)
                dno = rb.forward_response(prob, tro, approx, rb.ShiftedFactorCache()).data
                miso = 0.5 * float(np.sum((W * (dno - data.d_obs)) ** 2))
                rvo, _ = rb.reg_value_grad(reg, tro)
                sec.append((np.sqrt(r1o @ r1o + r2o @ r2o), miso + lam * rvo))
            out[f"secfloor_{k}"] = np.array(max(abs(sec[0][0] - sec[1][0]) / sec[0][0],
                                                abs(sec[0][1] - sec[1][1]) / sec[0][1]))
            print(f"k={k}: phi {float(out[f'phi_{k}']):.6e} floor {floor:.2e} "
                  f"{time.time() - t:.1f}s", flush=True)
    rr = np.random.default_rng(7)
    u = rr.standard_normal(P)
    y = rr.standard_normal(R.shape[0])
    out.update(R_u=R @ u, R_t_y=R.T @ y, R_nnz=np.array(R.nnz),
               R_sha=np.array(hashlib.sha256(np.ascontiguousarray(R.data).tobytes()
                                             + np.ascontiguousarray(R.indices).tobytes()
                                             ).hexdigest()))
    np.savez_compressed(os.path.join(HERE, fname), **out)
    print(f"{fname}: N {prob.dof_count} P {P} adjoint {float(out['adjoint']):.2e} "
          f"{time.time() - t:.1f}s")


def golden_rundir():
    from rundir_case import rundir_case
    """The reference's own write_run_artifacts (reporting.py:139-187) on a
    synthetic state: the committed files pin the rundir format."""
    import scipy.sparse as sp
    c = rundir_case()
    state = rb.InversionState(model=rb.Model(c["m"], c["m_ref"]), lam=c["lam"], nu=c["nu"],
                              phi=c["phi"], chi2=c["chi2"],
                              history=[rb.inversion.IterationRecord(**h) for h in c["history"]],
                              diagnostic=c["diagnostic"], counters=c["counters"])
    data = rb.DataSet(d_obs=c["d_obs"], sigma_d=c["sigma"], times=c["times"],
                      receivers=np.zeros((c["M_r"], 2)), eps_r=0.0, eps_a=1.0, seed=0,
                      provenance={})

    class _P:
        receiver_count = c["M_r"]
        Q = sp.csr_matrix((c["M_r"], 1))

    class _A:
        channels = rb.TimeChannels(c["times"])
    out = os.path.join(HERE, "rundir_ref")
    rb.reporting.write_run_artifacts(out, state, data, _P(), _A(), c["d_pred"])
    print("rundir_ref:", sorted(os.listdir(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c1", action="store_true")
    ap.add_argument("--c1true", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    if args.only == "rundir":
        golden_rundir()
        return
    if args.only == "c1true":
        golden_c1_true(fit_approximants()["C1"])
        return
    approxes = fit_approximants()
    golden_2d()
    golden_3d("C1", 6, approxes["C1"], "ref3d_n6.npz")
    golden_3d("C3", 6, approxes["C3"], "ref3d_c3_n6.npz", lsqr_iters=(1, 3))
    if args.c1:
        golden_3d("C1", 16, approxes["C1"], "ref3d_C1.npz", lsqr_iters=(1, 3, 5, 20))
    if args.c1true:
        golden_c1_true(approxes["C1"])


if __name__ == "__main__":
    main()
