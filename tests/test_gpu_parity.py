"""GPU parity: the device path (libdrba.so through the C ABI) against golden
vectors from the unmodified reference and against the CPU oracle.

Tolerances (BASELINE north_star): forward data <= 1e-9, J v / J^T w <= 1e-8
relative; GN update dm judged against the reference's own solver-to-solver
floor: <= 1e-8 where that floor is below 1e-10 (<= 5 LSQR
iterations), else within 10x of the floor measured here on the same inputs.
"""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from conftest import golden, rel
import paper_2605_19951_b200 as rb
from paper_2605_19951_b200.engine import Engine
from oracle import rbainv_oracle as orc

pytestmark = pytest.mark.gpu


def _model(prob, m):
    return rb.Model(np.asarray(m, dtype=float), np.asarray(m, dtype=float))


def _data(z):
    return rb.DataSet(d_obs=z["d_obs"], sigma_d=z["sigma_d"], times=np.zeros(1),
                      receivers=np.zeros((1, 3)), eps_r=0.0, eps_a=1.0, seed=0, provenance={})


@pytest.mark.parametrize("fname,name", [("ref3d_n6.npz", "C1"), ("ref3d_c3_n6.npz", "C3")])
def test_forward_jvp_vjp_vs_reference(gpu, fname, name):
    z = golden(fname)
    prob, _ = rb.build_config(name, n=int(z["n"]))
    approx = rb.config_approximant(name)
    model = _model(prob, z["m"])
    cache = rb.ShiftedFactorCache()
    d = rb.forward_response(prob, model, approx, cache).data
    assert rel(d, z["d"]) <= 1e-9
    opr = rb.JacobianOperator(prob, model, approx, cache)
    assert rel(opr.jvp(z["v"]), z["jv"]) <= 1e-8
    assert rel(opr.vjp(z["w"]), z["jtw"]) <= 1e-8
    assert rb.adjoint_test(opr, trials=3, seed=4) <= 1e-8


def test_gn_update_vs_reference_n6(gpu):
    z = golden("ref3d_n6.npz")
    prob, _ = rb.build_config("C1", n=6)
    approx = rb.config_approximant("C1")
    model = _model(prob, z["m"])
    cache = rb.ShiftedFactorCache()
    reg = rb.build_reg(prob.grid, root="chol")
    opr = rb.JacobianOperator(prob, model, approx, cache)
    data = _data(z)
    from paper_2605_19951_b200.inversion import _augmented_lsqr
    for k in (1, 3, 5):
        dm, itn, _ = _augmented_lsqr(opr, reg, data, z["d"], model, float(z["lam"]),
                                     rb.LsqrConfig(tol=0.0, max_iters=k))
        assert itn == int(z[f"itn_{k}"])
        floor, _ = orc.lsqr_floor(prob, z["m"], approx.poles, approx.residues, reg.R_factor,
                                  1.0 / z["sigma_d"], z["d_obs"], float(z["lam"]), k)
        err = rel(dm, z[f"dm_{k}"])
        print(f"GN update after {k} LSQR its: gpu-vs-ref {err:.2e}, ref floor {floor:.2e}")
        assert err <= max(1e-8, 10 * floor), (k, err, floor)


def test_c1_full_size_vs_reference(gpu):
    """BASELINE config 1 at full size (n=16, N=26,416, 8 poles)."""
    z = golden("ref3d_C1.npz")
    prob, _ = rb.build_config("C1", n=16)
    approx = rb.config_approximant("C1")
    model = _model(prob, z["m"])
    cache = rb.ShiftedFactorCache()
    d = rb.forward_response(prob, model, approx, cache).data
    assert rel(d, z["d"]) <= 1e-9
    opr = rb.JacobianOperator(prob, model, approx, cache)
    assert rel(opr.jvp(z["v"]), z["jv"]) <= 1e-8
    assert rel(opr.vjp(z["w"]), z["jtw"]) <= 1e-8
    reg = rb.build_reg(prob.grid, root="chol")
    from paper_2605_19951_b200.inversion import _augmented_lsqr
    dm, itn, _ = _augmented_lsqr(opr, reg, _data(z), z["d"], model, float(z["lam"]),
                                 rb.LsqrConfig(tol=0.0, max_iters=5))
    assert itn == 5
    # reference floor at C1 is ~1e-9 after 5 iterations
    err = rel(dm, z["dm_5"])
    print(f"C1 GN update (5 its): gpu-vs-ref {err:.2e}")
    assert err <= 1e-7


@pytest.mark.parametrize("air", [False, True])
def test_solves_vs_splu_and_transpose(gpu, air):
    """Random complex RHS.  Without air the reference's residual bound
    (shifted.py:193-196) applies; with 1e-8 S/m air cells A is nearly singular
    on the gradient null space (cond ~ 1e17), so the check is the normwise
    backward error, which splu meets at the same level."""
    prob, _ = rb.build_config("C1", n=8)
    approx = rb.config_approximant("C1")
    model = prob.true_model() if air else rb.Model(np.full(prob.grid.cell_count, np.log(0.01)),
                                                   np.full(prob.grid.cell_count, np.log(0.01)))
    cache = rb.ShiftedFactorCache()
    rb.factorize_all_poles(prob, model, approx, cache)
    M = orc.assemble_M(prob, model.m)
    rng = np.random.default_rng(5)
    b = rng.standard_normal(prob.dof_count) + 1j * rng.standard_normal(prob.dof_count)
    for i in (0, 3, 7):
        A = (prob.K.astype(complex) - approx.poles[i] * M.astype(complex)).tocsc()
        x = cache.solve(i, b)
        xt = cache.solve(i, b, trans="T")
        xs = spla.splu(A).solve(b)
        res = np.linalg.norm(A @ x - b)
        nA = abs(A).sum(axis=1).max()
        bwd = res / (nA * np.linalg.norm(x) + np.linalg.norm(b))
        bwd_s = np.linalg.norm(A @ xs - b) / (nA * np.linalg.norm(xs) + np.linalg.norm(b))
        print(f"pole {i} air={air}: residual {res / np.linalg.norm(b):.2e}, backward {bwd:.2e}"
              f" (splu {bwd_s:.2e}), vs splu {rel(x, xs):.2e}")
        assert bwd <= max(1e-15, 10 * bwd_s)
        if not air:
            assert res / np.linalg.norm(b) <= 1e-8
            assert rel(x, xs) <= 1e-9
        np.testing.assert_array_equal(x, xt)
        # repeat solves are bitwise identical (deterministic kernels)
        np.testing.assert_array_equal(x, cache.solve(i, b))
        # multi-RHS solve agrees column by column
        B = np.stack([b, b.conj(), 2 * b], axis=1)
        X = cache.solve(i, B)
        assert rel(X[:, 0], x) <= 1e-14 and rel(X[:, 2], 2 * x) <= 1e-14


def test_counters_and_cache_semantics(gpu):
    prob, _ = rb.build_config("C1", n=4)
    approx = rb.config_approximant("C1")
    model = prob.reference_model()
    cache = rb.ShiftedFactorCache()
    m = approx.pole_count
    rb.solve_all_poles(prob, model, approx, prob.f, cache)
    assert cache.counters.factorizations == m and cache.counters.solves == m
    rb.solve_all_poles(prob, model, approx, prob.f, cache)
    assert cache.counters.factorizations == m
    opr = rb.JacobianOperator(prob, model, approx, cache)
    s0 = cache.counters.solves
    opr.jvp(np.ones(opr.shape[1]))
    assert cache.counters.solves - s0 == m
    opr.vjp(np.ones(opr.shape[0]))
    assert cache.counters.solves - s0 == 2 * m
    cache.activate("someone-else")
    with pytest.raises(RuntimeError):
        opr.jvp(np.ones(opr.shape[1]))
    with pytest.raises(rb.CacheMissError):
        cache.solve(0, np.zeros(prob.dof_count, complex))


def test_generic_cache_with_reference_2d_problem(gpu):
    """Generic mode: factorize(i, A) with assembled SciPy matrices of the
    reference's 2-D fixture; solutions vs the reference's own g."""
    z = golden("ref2d_small.npz")
    N = z["K_indptr"].size - 1
    K = sp.csr_matrix((z["K_data"], z["K_indices"], z["K_indptr"]), shape=(N, N))

    class P:
        pass
    p = P()
    p.K, p.cell_dofs, p.mass_local, p._scatter = K, z["cell_dofs"], z["mass_local"], None
    M = orc.assemble_M(p, z["m"]).astype(complex)
    cache = rb.ShiftedFactorCache()
    cache.activate("tag")
    for i, xi in enumerate(z["poles"]):
        cache.factorize(i, (K.astype(complex) - xi * M).tocsc())
    g = np.array([cache.solve(i, z["f"]) for i in range(z["poles"].size)])
    assert rel(g, z["g"][:, :, 0]) <= 1e-10
    assert cache.counters.factorizations == z["poles"].size


def test_scalar_shifted_inverse_kat(gpu):
    """test_shifted.py:26-36: one dof, A = k - xi mu."""
    k, mu = 2.0, 2.0 / 3.0
    cache = rb.ShiftedFactorCache()
    cache.activate("t")
    for i, xi in enumerate([0.5 + 1.5j, -2.0 + 3.0j]):
        cache.factorize(i, sp.csr_matrix(np.array([[k - xi * mu]])))
        g = cache.solve(i, np.array([1.0]))
        assert abs(g[0] - 1.0 / (k - xi * mu)) <= 1e-14 * abs(1.0 / (k - xi * mu))


def test_singular_shift_raises(gpu):
    """test_shifted.py:170-177: an exactly singular shift -> SolveError."""
    cache = rb.ShiftedFactorCache()
    cache.activate("t")
    with pytest.raises(rb.SolveError):
        cache.factorize(0, sp.csr_matrix(np.array([[0.0 + 0.0j]])))


def test_scaling_benchmark_checksums_bitwise(gpu):
    """reporting.scaling_benchmark (the C2 harness template, reporting.py:87-122):
    W pole shards (emulated ranks on one device) give bit-identical pole
    solutions for W = 1, 2, 4, 8 (test_acceptance.py:212-234), and each
    shard's factorisation gets faster as it owns fewer poles."""
    prob, _ = rb.build_config("C1", n=8)
    approx = rb.config_approximant("C1")
    rows = rb.scaling_benchmark(prob, prob.true_model(), approx, worker_counts=(1, 2, 4, 8),
                                solve_repeats=2)
    assert len({r["checksum"] for r in rows}) == 1
    assert all(r["emulated"] and r["factorize_ms"] > 0 and r["solve_ms"] > 0 for r in rows)
    assert rows[0]["efficiency"] == pytest.approx(1.0)


def test_taylor_slopes_device(gpu):
    """sensitivity.py:135-172 / test_sensitivity.py:166-174 on the device path."""
    prob, _ = rb.build_config("C1", n=6)
    approx = rb.config_approximant("C1")
    m = np.where(prob.m_true < np.log(1e-6), np.log(0.01), prob.m_true)
    model = rb.Model(m, m)
    rng = np.random.default_rng(1)
    direction = rng.standard_normal(prob.grid.cell_count)
    direction /= np.max(np.abs(direction))
    rep = rb.taylor_test(prob, model, approx, direction, [1e-1, 1e-2, 1e-3, 1e-4])
    assert 0.9 <= rep.slope0 <= 1.1
    assert 1.8 <= rep.slope1 <= 2.2


def test_run_inversion_matches_oracle_first_iteration(gpu):
    """One full GN iteration of run_inversion (gradient, 5 LSQR its, Armijo
    line search with refactorisations) against the oracle's restatement on the
    same inputs: same accepted step and objective to tolerance."""
    z = golden("ref3d_n6.npz")
    prob, _ = rb.build_config("C1", n=6)
    approx = rb.config_approximant("C1")
    data = _data(z)
    reg = rb.build_reg(prob.grid, root="chol")
    cfg = rb.InversionConfig(lambda0=float(z["lam"]), max_gn=1, chi2_target=0.0,
                             lsqr=rb.LsqrConfig(tol=0.0, max_iters=5), m0=z["m"])
    prob.sigma_background = float(np.exp(z["m"][0]))
    st = rb.run_inversion(prob, data, approx, cfg, reg=reg)
    rec = st.history[0]
    # oracle: same iteration by hand
    fac = orc.PoleFactors()
    m0 = z["m"]
    W = 1.0 / z["sigma_d"]
    d0, g = orc.forward_response(prob, m0, approx.poles, approx.residues, fac)
    J = orc.Jacobian(prob, m0, approx.poles, approx.residues, fac, g=g)
    dm, _, _ = orc.augmented_lsqr(J, reg.R_factor, W, z["d_obs"], d0, m0, m0,
                                  float(z["lam"]), 0.0, 5)
    def phi(mm):
        d, _ = orc.forward_response(prob, mm, approx.poles, approx.residues, orc.PoleFactors())
        r = mm - m0
        return 0.5 * float(np.sum((W * (d - z["d_obs"])) ** 2)) + float(z["lam"]) * 0.5 * float(r @ (reg.L @ r))
    phi0 = phi(m0)
    grad = J.vjp(W * W * (d0 - z["d_obs"]))
    slope = float(grad @ dm)
    eta, ok, phi_acc, n = orc.line_search(phi0, slope, lambda e: phi(m0 + e * dm))
    assert rec.accepted == ok and rec.phi_evals == n
    assert abs(rec.eta - eta) <= 1e-6 * max(1.0, abs(eta))
    assert abs(rec.phi - phi_acc) <= 1e-6 * abs(phi_acc)
    assert abs(rec.directional_slope - slope) <= 1e-6 * abs(slope)


def test_eight_rhs_solves_vs_splu(gpu):
    """8 right-hand sides per sweep (C5 has 8 sources): the NR = 8 kernels,
    including the two-column-pass backward with the dependent block handled
    last, agree with SuperLU column by column (n = 10: fronts of up to 5
    pivot blocks)."""
    prob, _ = rb.build_config("C5", n=10)
    approx = rb.config_approximant("C5")
    m0 = np.full(prob.grid.cell_count, np.log(0.01))
    model = rb.Model(m0, m0)
    cache = rb.ShiftedFactorCache()
    rb.factorize_all_poles(prob, model, approx, cache)
    assert cache.engine.S == 8
    M = orc.assemble_M(prob, model.m)
    rng = np.random.default_rng(8)
    B = rng.standard_normal((prob.dof_count, 8)) + 1j * rng.standard_normal((prob.dof_count, 8))
    for i in (0, 11):
        A = (prob.K.astype(complex) - approx.poles[i] * M.astype(complex)).tocsc()
        X = cache.solve(i, B)
        Xs = spla.splu(A).solve(B)
        err = max(rel(X[:, k], Xs[:, k]) for k in range(8))
        print(f"pole {i}: 8-RHS solve vs splu {err:.2e}")
        assert err <= 1e-9


@pytest.mark.parametrize("mode", ["0", "1", "2"])
def test_four_rhs_backward_kernels(gpu, monkeypatch, mode):
    """4 right-hand sides (C3/C4's 4 sources): the backward sweep's variants --
    scalar kernels (RBA_BWD_MMA=0), FP64 tensor-core kernel for the small
    fronts (1, default) and for the large fronts too (2) -- all agree with
    SuperLU column by column (n = 12 with air layers: fronts of several pivot
    blocks, borders longer than one shared-memory chunk are covered by the C4
    tests)."""
    monkeypatch.setenv("RBA_BWD_MMA", mode)
    prob, _ = rb.build_config("C4", n=12)
    approx = rb.config_approximant("C4")
    model = rb.Model(prob.m_true, prob.m_true)
    cache = rb.ShiftedFactorCache()
    rb.factorize_all_poles(prob, model, approx, cache)
    assert cache.engine.S == 4
    M = orc.assemble_M(prob, model.m)
    rng = np.random.default_rng(4)
    B = rng.standard_normal((prob.dof_count, 4)) + 1j * rng.standard_normal((prob.dof_count, 4))
    for i in (0, 9):
        A = (prob.K.astype(complex) - approx.poles[i] * M.astype(complex)).tocsc()
        X = cache.solve(i, B)
        r = max(np.linalg.norm(A @ X[:, k] - B[:, k]) /
                (abs(A).sum(axis=1).max() * np.linalg.norm(X[:, k]) + np.linalg.norm(B[:, k])) for k in range(4))
        print(f"RBA_BWD_MMA={mode} pole {i}: normwise backward error {r:.2e}")
        assert r <= 1e-15           # (with 1e-8 S/m air the forward error is cond(A) x this)
    cache.engine.close()


def _c1_true():
    z = golden("ref3d_C1_true.npz")
    prob, _ = rb.build_config("C1", n=int(z["n"]))
    approx = rb.config_approximant("C1")
    model = rb.Model(z["m"], z["m_ref"])
    return z, prob, approx, model


def test_c1_true_model_forward_and_jacobian(gpu):
    """C1 at full size at its TRUE model: 1e-8 S/m air, 1 S/m block
    (make_golden.py golden_c1_true, unmodified reference)."""
    z, prob, approx, model = _c1_true()
    assert np.unique(np.exp(z["m"])).size >= 3           # air, half-space, block
    cache = rb.ShiftedFactorCache()
    d = rb.forward_response(prob, model, approx, cache).data
    opr = rb.JacobianOperator(prob, model, approx, cache)
    ef, ej, et = rel(d, z["d"]), rel(opr.jvp(z["v"]), z["jv"]), rel(opr.vjp(z["w"]), z["jtw"])
    adj = rb.adjoint_test(opr, trials=3, seed=4)
    print(f"C1 true model: forward {ef:.2e}  J v {ej:.2e}  J^T w {et:.2e}  adjoint {adj:.2e} "
          f"(reference {float(z['adjoint']):.2e})")
    assert ef <= 1e-9 and ej <= 1e-8 and et <= 1e-8
    assert adj <= 1e-8
    # the reference's d_clean of the old start-model golden is this same forward
    z0 = golden("ref3d_C1.npz")
    assert rel(d, z0["d_clean"]) <= 1e-9


def test_c1_true_model_gn_update(gpu):
    """GN update dm after 1/3/5/20 LSQR iterations at the true model with the
    reference's LAPACK R: <= max(1e-8, 10 x the reference's own solver-to-
    solver floor) (floors measured by make_golden.py), and the
    iteration-count-robust secondaries after the 20-iteration step."""
    import hashlib
    from paper_2605_19951_b200.inversion import _augmented_lsqr
    z, prob, approx, model = _c1_true()
    reg = rb.build_reg(prob.grid, root="chol")
    R = reg.R_factor
    rr = np.random.default_rng(7)
    u = rr.standard_normal(R.shape[1])
    y = rr.standard_normal(R.shape[0])
    same = hashlib.sha256(np.ascontiguousarray(R.data).tobytes() +
                          np.ascontiguousarray(R.indices).tobytes()).hexdigest() == str(z["R_sha"])
    print(f"reference R: bitwise {'identical' if same else 'different'}, R u {rel(R @ u, z['R_u']):.1e},"
          f" R^T y {rel(R.T @ y, z['R_t_y']):.1e}")
    assert R.nnz == int(z["R_nnz"])
    assert rel(R @ u, z["R_u"]) <= 1e-13 and rel(R.T @ y, z["R_t_y"]) <= 1e-13
    cache = rb.ShiftedFactorCache()
    opr = rb.JacobianOperator(prob, model, approx, cache)
    data = _data(z)
    lam = float(z["lam"])
    W = data.weights
    for k in (1, 3, 5, 20):
        dm, itn, _ = _augmented_lsqr(opr, reg, data, z["d"], model, lam,
                                     rb.LsqrConfig(tol=0.0, max_iters=k))
        assert itn == k
        err = rel(dm, z[f"dm_{k}"])
        floor = float(z[f"floor_{k}"]) if f"floor_{k}" in z else 0.0
        r1 = W * (opr.jvp(dm) + z["d"] - z["d_obs"])
        r2 = np.sqrt(lam) * (R @ (dm + model.m - model.m_ref))
        lin = float(np.sqrt(r1 @ r1 + r2 @ r2))
        elin = abs(lin - float(z[f"linres_{k}"])) / float(z[f"linres_{k}"])
        msg = f"k={k}: dm vs reference {err:.2e} (floor {floor:.2e}), linearised residual {elin:.1e}"
        if k in (5, 20):
            trial = rb.Model(model.m + dm, model.m_ref)
            dn = rb.forward_response(prob, trial, approx, rb.ShiftedFactorCache()).data
            mis = 0.5 * float(np.sum((W * (dn - z["d_obs"])) ** 2))
            rv, _ = rb.reg_value_grad(reg, trial)
            ephi = abs(mis + lam * rv - float(z[f"phi_{k}"])) / float(z[f"phi_{k}"])
            echi = abs(2 * mis / dn.size - float(z[f"chi2_{k}"])) / float(z[f"chi2_{k}"])
            msg += f", phi after step {ephi:.1e}, chi2 {echi:.1e}"
        # the reference's own secondaries floor (SuperLU COLAMD vs MMD_AT_PLUS_A,
        # same inputs) where the golden carries it, else the dm floor
        sec = float(z[f"secfloor_{k}"]) if f"secfloor_{k}" in z else floor
        msg += f" (secondaries floor {sec:.1e})"
        print(msg)
        assert err <= max(1e-8, 10 * floor), msg
        assert elin <= max(1e-8, 10 * sec), msg
        if k in (5, 20):
            assert ephi <= max(1e-8, 10 * sec) and echi <= max(1e-8, 10 * sec), msg


@pytest.mark.parametrize("air", [False, True])
def test_device_mass_assembly_vs_assemble_M(gpu, air):
    """K1 (k_exp + k_assemble_M, the device gather of sum_c e^{m_c} M_c) against
    the oracle's COO->CSR assemble_M (mesh.py:348-355), entry by entry on the
    lower-triangle pattern, at the true model with 1e-8 S/m air and at the
    homogeneous start model; K against problem.K."""
    prob, _ = rb.build_config("C1", n=10)
    m = prob.m_true if air else np.full(prob.m_true.shape, np.log(0.01))
    eng = Engine(prob, None)
    eng.set_model(m)
    rows, cols, Kv, Mv = eng.pattern(with_M=True)
    M = orc.assemble_M(prob, m).tocsr()
    Mref = np.asarray(M[rows, cols]).ravel()
    Kref = np.asarray(prob.K.tocsr()[rows, cols]).ravel()
    assert np.all(rows >= cols) and np.count_nonzero(Mref) == sp.tril(M).count_nonzero()
    scale = np.abs(Mref).max()
    assert np.abs(Mv - Mref).max() <= 1e-14 * scale
    np.testing.assert_allclose(Kv, Kref, rtol=0, atol=1e-14 * np.abs(Kref).max())
    eng.close()
