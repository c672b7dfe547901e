"""At-size verification of the pivot-free complex-symmetric LDL^T and of the
operators built on it (VERDICT r1 "verify the problem you benchmark"):

* normwise backward error |A_i x - b| / (|A_i| |x| + |b|) of every pole at C2
  size (n = 32, N = 220,256, random sigma), computed with a host SciPy SpMV of
  the oracle's assemble_M (mesh.py:348-355) -- the reference's residual guard
  is shifted.py:193-196;
* the same at the C4 shape (1e-8 S/m air) against SuperLU's own backward
  error on the same matrices;
* growth max|L'|^2 / max|A| and the smallest pivot of the factor;
* C3 at size (n = 32, 4 sources x 100 receivers): adjointness
  (sensitivity.py:175-188) <= 1e-8;
* emulated multi-GPU (G engines on one device, each owning poles i mod G):
  forward data, J v and J^T w bitwise equal to G = 1 (test_acceptance.py:
  212-234 worker-count invariance);
* trans 'H', pole_solutions, generic-mode memory, rejected line search.
"""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla
import torch

from conftest import rel
import paper_2605_19951_b200 as rb
from paper_2605_19951_b200 import _lib
from paper_2605_19951_b200._lib import ptr
from paper_2605_19951_b200.engine import Engine
from paper_2605_19951_b200.parallel import PoleComm, ShardComm, gathered_slot_of_pole
from oracle import rbainv_oracle as orc

pytestmark = pytest.mark.gpu


def _A(prob, m, xi):
    return (prob.K.astype(complex) - xi * orc.assemble_M(prob, m).astype(complex)).tocsr()


def _bwd(A, x, b):
    nA = abs(A).sum(axis=1).max()
    return float(np.linalg.norm(A @ x - b) / (nA * np.linalg.norm(x) + np.linalg.norm(b)))


def _growth(eng, slot, A):
    st = eng.factor_stats(slot)
    amax = float(abs(A).max())
    return st["max_abs_Lp"] ** 2 / amax, st["min_abs_sqrt_d"] ** 2 / amax, st


def test_c2_size_backward_error_all_poles(gpu):
    """BASELINE config 2 at full size: all 16 poles, random sigma in [1e-3, 1]."""
    prob, _ = rb.build_config("C2")
    approx = rb.config_approximant("C2")
    rng = np.random.default_rng(11)
    b = rng.standard_normal(prob.dof_count) + 1j * rng.standard_normal(prob.dof_count)
    eng = Engine(prob, None)
    eng.set_sources(b[None, :])
    eng.set_poles(approx)
    eng.set_model(prob.m_true)
    eng.factor()
    worst = 0.0
    for i in range(approx.pole_count):
        A = _A(prob, prob.m_true, approx.poles[i])
        x = eng.solve(i, b)
        e = _bwd(A, x, b)
        gr, dmin, st = _growth(eng, i, A)
        print(f"C2 pole {i:2d} xi={approx.poles[i]:.3e}: backward {e:.2e} growth {gr:.2e} "
              f"min|d|/max|A| {dmin:.2e}")
        assert st["nonfinite"] == 0
        assert gr < 1e3
        worst = max(worst, e)
    assert worst <= 1e-14, worst
    eng.close()


def test_c4_shape_backward_error_vs_superlu(gpu):
    """C4 shape (6 air layers at 1e-8 S/m, dipping plate) at n = 12: every
    pole's backward error within 10x of SuperLU's on the same matrix."""
    prob, _ = rb.build_config("C4", n=12)
    approx = rb.config_approximant("C4")
    rng = np.random.default_rng(12)
    b = rng.standard_normal(prob.dof_count) + 1j * rng.standard_normal(prob.dof_count)
    eng = Engine(prob, None)
    eng.set_sources(b[None, :])
    eng.set_poles(approx)
    eng.set_model(prob.m_true)
    eng.factor()
    for i in range(approx.pole_count):
        A = _A(prob, prob.m_true, approx.poles[i])
        e = _bwd(A, eng.solve(i, b), b)
        es = _bwd(A, spla.splu(A.tocsc()).solve(b), b)
        gr, dmin, _ = _growth(eng, i, A)
        print(f"C4-shape pole {i:2d}: backward {e:.2e} (SuperLU {es:.2e}) growth {gr:.2e} "
              f"min|d|/max|A| {dmin:.2e}")
        assert e <= max(10 * es, 1e-15), (i, e, es)
    eng.close()


def test_c3_size_adjointness(gpu):
    """BASELINE config 3 at full size (n = 32, 4 loops, 10x10 receivers,
    31 times, 16 poles): <Jv, w> = <v, J^T w> to 1e-8 (reference metric)."""
    prob, _ = rb.build_config("C3")
    approx = rb.config_approximant("C3")
    cache = rb.ShiftedFactorCache()
    opr = rb.JacobianOperator(prob, prob.true_model(), approx, cache)
    worst = rb.adjoint_test(opr, trials=5, seed=0)
    rng = np.random.default_rng(1)
    v = rng.standard_normal(opr.shape[1])
    w = rng.standard_normal(opr.shape[0])
    jv, jtw = opr.jvp(v), opr.vjp(w)
    nw = abs(jv @ w - v @ jtw) / (np.linalg.norm(jv) * np.linalg.norm(w))
    print(f"C3 adjointness: reference metric {worst:.2e}, normwise {nw:.2e}")
    assert worst <= 1e-8
    assert nw <= 1e-12


_EmulatedComm = ShardComm     # rank r of a G-rank job; the test exchanges the partials


@pytest.mark.parametrize("green", [True, False])
def test_emulated_multi_gpu_bitwise(gpu, green):
    """G in {2, 3, 8}: G engines on one device, engine r owning poles i mod G
    (per-rank Engine, gathered slot map, device combine); forward data, J v
    and J^T w must equal the single-engine result bit for bit."""
    prob, _ = rb.build_config("C3", n=8)
    approx = rb.config_approximant("C3")
    m = prob.m_true
    rng = np.random.default_rng(2)
    v = torch.as_tensor(rng.standard_normal(prob.grid.cell_count), device="cuda")
    w = torch.as_tensor(rng.standard_normal(prob.source_count * approx.channels.count *
                                            prob.receiver_count), device="cuda")

    def run(G):
        engs = [Engine(prob, approx, comm=_EmulatedComm(G, r) if G > 1 else PoleComm(1, 0))
                for r in range(G)]
        for e in engs:
            if not green:
                e.set_option("green", 0)
            e.set_model(m)
            e.factor()
        som = gathered_slot_of_pole(approx.pole_count, G) if G > 1 else engs[0].slot_of_pole
        outs = []
        for kind in ("fwd", "jvp", "vjp"):
            parts = []
            for e in engs:
                if kind == "fwd":
                    _lib.check(e.lib.rba_forward_partial(e.ctx, ptr(e.qpart)))
                    parts.append(e.qpart.clone())
                elif kind == "jvp":
                    _lib.check(e.lib.rba_jvp_partial(e.ctx, ptr(v), ptr(e.qpart)))
                    parts.append(e.qpart.clone())
                else:
                    _lib.check(e.lib.rba_vjp_partial(e.ctx, ptr(w), ptr(e.tpart)))
                    parts.append(e.tpart.clone())
            allp = torch.cat(parts, 0).contiguous()
            e0 = engs[0]
            if kind == "vjp":
                out = torch.empty(e0.P, dtype=torch.float64, device="cuda")
                _lib.check(e0.lib.rba_combine_cells(e0.ctx, ptr(allp), ptr(som), ptr(out)))
            else:
                out = torch.empty(e0.S * e0.Kt * e0.Mr, dtype=torch.float64, device="cuda")
                _lib.check(e0.lib.rba_combine_data(e0.ctx, ptr(allp), ptr(som),
                                                   1 if kind == "jvp" else 0, ptr(out)))
            outs.append(out.cpu().numpy())
        assert all(bool(e.info()["green"]) == green for e in engs)
        for e in engs:
            e.close()
        return outs

    ref = run(1)
    for G in (2, 3, 8):
        got = run(G)
        for kind, a, b in zip(("forward", "J v", "J^T w"), got, ref):
            np.testing.assert_array_equal(a, b, err_msg=f"G={G} {kind}")


def test_trans_h_and_invalid(gpu):
    """_Factor.solve(rhs, trans) (shifted.py:58-61): 'H' solves A^H x = b."""
    prob, _ = rb.build_config("C1", n=6)
    approx = rb.config_approximant("C1")
    cache = rb.ShiftedFactorCache()
    rb.factorize_all_poles(prob, prob.true_model(), approx, cache)
    A = _A(prob, prob.true_model().m, approx.poles[2])
    rng = np.random.default_rng(3)
    b = rng.standard_normal(prob.dof_count) + 1j * rng.standard_normal(prob.dof_count)
    xh = cache.solve(2, b, trans="H")
    assert _bwd(A.conj().T.tocsr(), xh, b) <= 1e-14
    np.testing.assert_array_equal(xh, np.conj(cache.solve(2, np.conj(b))))
    with pytest.raises(ValueError):
        cache.solve(2, b, trans="X")


def test_pole_solutions_are_used(gpu):
    """JacobianOperator(..., pole_solutions=g) contracts dM with the given g
    (sensitivity.py:43-59): J is linear in g, so 2g doubles J v and J^T w."""
    prob, _ = rb.build_config("C1", n=6)
    approx = rb.config_approximant("C1")
    model = prob.true_model()
    cache = rb.ShiftedFactorCache()
    g = rb.solve_all_poles(prob, model, approx, prob.f, cache)
    o1 = rb.JacobianOperator(prob, model, approx, cache, pole_solutions=g)
    rng = np.random.default_rng(4)
    v = rng.standard_normal(o1.shape[1])
    w = rng.standard_normal(o1.shape[0])
    jv, jtw = o1.jvp(v), o1.vjp(w)
    o2 = rb.JacobianOperator(prob, model, approx, cache, pole_solutions=2 * g)
    assert rel(o2.jvp(v), 2 * jv) <= 1e-14
    assert rel(o2.vjp(w), 2 * jtw) <= 1e-14


def test_generic_mode_allocates_per_pole(gpu):
    """cache.factorize(i, A) allocates factor storage for the poles it sees,
    not for max_poles (32 slots at C4 would need 269 GB)."""
    z = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden",
                                           "ref2d_small.npz"))
    N = z["K_indptr"].size - 1
    K = sp.csr_matrix((z["K_data"], z["K_indices"], z["K_indptr"]), shape=(N, N))
    cache = rb.ShiftedFactorCache(max_poles=32)
    cache.activate("t")
    for i in range(2):
        cache.factorize(i, (K - (1.0 + 1j * (i + 1)) * sp.eye(N)).tocsc())
    info = cache.engine.info()
    per = info["mem_factor"] // 2
    assert per > 0
    cache.factorize(5, (K - 3j * sp.eye(N)).tocsc())
    assert cache.engine.info()["mem_factor"] == 3 * per


def test_rejected_line_search_continues(gpu, monkeypatch):
    """after a rejected line search the reference raises "cache
    has moved" in the next iteration (inversion.py:248,257-263).  Here the
    next iteration re-activates the current model (m refactorisations) and
    continues; its update equals a fresh GN step at that model."""
    import paper_2605_19951_b200.inversion as inv
    z = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden",
                                           "ref3d_n6.npz"))
    prob, _ = rb.build_config("C1", n=6)
    approx = rb.config_approximant("C1")
    data = rb.DataSet(d_obs=z["d_obs"], sigma_d=z["sigma_d"], times=np.zeros(1),
                      receivers=np.zeros((1, 3)), eps_r=0.0, eps_a=1.0, seed=0, provenance={})
    reg = rb.build_reg(prob.grid, root="chol")
    real_ls = inv.line_search
    calls = []

    def ls(phi0, slope, ev, **kw):
        calls.append(1)
        if len(calls) == 1:              # evaluate two trials, then reject
            ev(1.0)
            ev(0.5)
            return inv.LineSearchResult(2.0 ** -6, False, phi0, 2)
        return real_ls(phi0, slope, ev, **kw)

    monkeypatch.setattr(inv, "line_search", ls)
    cfg = rb.InversionConfig(lambda0=float(z["lam"]), max_gn=2, chi2_target=0.0,
                             lsqr=rb.LsqrConfig(tol=0.0, max_iters=3), m0=z["m"])
    st = rb.run_inversion(prob, data, approx, cfg, reg=reg)
    assert len(st.history) == 2
    r1, r2 = st.history
    m = approx.pole_count
    assert not r1.accepted and r1.factorizations == 2 * m
    # iteration 2: the current model is refactorised once, then the trials
    assert r2.factorizations == m * (1 + r2.phi_evals)
    assert r2.lam == pytest.approx(r1.lam / 2)
    # the second update equals a fresh GN step at the unchanged model with lambda/2
    cache = rb.ShiftedFactorCache()
    model = rb.Model(z["m"], z["m"])
    opr = rb.JacobianOperator(prob, model, approx, cache)
    d0 = opr.engine.forward().cpu().numpy()
    dm, itn, _ = inv._augmented_lsqr(opr, reg, data, d0, model, r2.lam, cfg.lsqr)
    slope = float(opr.vjp(data.weights * data.weights * (d0 - data.d_obs)) @ dm)
    assert r2.directional_slope == pytest.approx(slope, rel=1e-9)


def test_device_reg_value_grad(gpu):
    """reg_value_grad (regularization.py:71-75) on the device SpMV of L."""
    from paper_2605_19951_b200.inversion import reg_value_grad_device
    prob, _ = rb.build_config("C1", n=6)
    reg = rb.build_reg(prob.grid)
    eng = Engine(prob, rb.config_approximant("C1"))
    rng = np.random.default_rng(5)
    m = rng.standard_normal(prob.grid.cell_count)
    mref = np.zeros_like(m)
    val, Lr = reg_value_grad_device(eng, reg, torch.as_tensor(m - mref, device="cuda"))
    v_h, g_h = rb.reg_value_grad(reg, rb.Model(m, mref))
    assert abs(val - v_h) <= 1e-13 * abs(v_h)
    assert rel(Lr.cpu().numpy(), g_h) <= 1e-14
    eng.close()
