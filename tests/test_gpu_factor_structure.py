"""Front-by-front parity of the device factor with the host emulation of the
same multifrontal algorithm (tests/mf_emulator.py)."""

import numpy as np
import pytest

from conftest import rel
import mf_emulator as mf
import paper_2605_19951_b200 as rb
from paper_2605_19951_b200 import _lib
from paper_2605_19951_b200._lib import ptr
from oracle import rbainv_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [4, 6, 8])
def test_device_fronts_match_emulation(gpu, n):
    prob, _ = rb.build_config("C1", n=n)
    approx = rb.config_approximant("C1")
    model = prob.true_model()
    cache = rb.ShiftedFactorCache()
    rb.factorize_all_poles(prob, model, approx, cache)
    eng = cache.engine
    S = mf.analyze(prob.K, prob.dof_coords, 64)
    tot = int(S["panel_off"][-1])
    buf = np.empty(tot, dtype=np.complex128)
    _lib.check(eng.lib.rba_get_factor(eng.ctx, 0, ptr(buf.view(np.float64)), tot))
    A = (prob.K.astype(complex) - approx.poles[0] * orc.assemble_M(prob, model.m)).tocsr()
    panels = mf.factor(A, S)
    worst = []
    for s, Lh in enumerate(panels):
        nf, p = S["nf"][s], S["npiv"][s]
        Ld = mf.device_panel_to_ldl(buf[S["panel_off"][s]:S["panel_off"][s] + nf * p].reshape(p, nf).T, p)
        mask = np.tril(np.ones((nf, p), bool))
        e = np.abs(Ld[mask] - Lh[mask]).max() / max(np.abs(Lh[mask]).max(), 1e-300)
        worst.append((float(e), s, int(p), int(nf), int(S["level"][s])))
    worst.sort(reverse=True)
    print("worst fronts (err, s, p, nf, level):", worst[:5])
    assert worst[0][0] <= 1e-10
    # the loop source (physical RHS): well conditioned observables
    b = prob.f.astype(complex)
    x = cache.solve(0, b)
    assert rel(prob.Q @ x, prob.Q @ mf.solve(b, panels, S)) <= 1e-10


def _worst_front_error(buf, panels, S):
    worst = 0.0
    for s, Lh in enumerate(panels):
        nf, p = S["nf"][s], S["npiv"][s]
        Ld = mf.device_panel_to_ldl(buf[S["panel_off"][s]:S["panel_off"][s] + nf * p].reshape(p, nf).T, p)
        mask = np.tril(np.ones((nf, p), bool))
        worst = max(worst, np.abs(Ld[mask] - Lh[mask]).max() / max(np.abs(Lh[mask]).max(), 1e-300))
    return float(worst)


def test_dmma_gemm_matches_dfma_reference(gpu, monkeypatch):
    """Every GEMM variant (the DFMA reference kernel with the substitution TRSM,
    the DMMA kernels v3..v8 with the inverted-diagonal TRSM) yields the host
    emulation's factor front by front (C1 shape, n=10: multi-block fronts),
    and the variants agree with one another."""
    prob, _ = rb.build_config("C1", n=10)
    approx = rb.config_approximant("C1")
    model = prob.true_model()
    S = mf.analyze(prob.K, prob.dof_coords, 64)
    A = (prob.K.astype(complex) - approx.poles[2] * orc.assemble_M(prob, model.m)).tocsr()
    panels = mf.factor(A, S)
    out = []
    modes = ("dfma", "v3", "v4", "v5", "v5b", "v6", "v6b", "v6c", "v6d", "v7", "v7b", "v8", "v8b", "v8c")
    for mode in modes:
        monkeypatch.setenv("RBA_GEMM", mode)
        cache = rb.ShiftedFactorCache()
        rb.factorize_all_poles(prob, model, approx, cache)
        eng = cache.engine
        tot = int(S["panel_off"][-1])
        buf = np.empty(tot, dtype=np.complex128)
        _lib.check(eng.lib.rba_get_factor(eng.ctx, 2, ptr(buf.view(np.float64)), tot))
        out.append(buf)
        eng.close()
        err = _worst_front_error(buf, panels, S)
        print(f"GEMM {mode}: worst front vs emulation {err:.2e}, factor vs DFMA {rel(buf, out[0]):.2e}")
        assert err <= 1e-10, mode
    for mode, o in zip(modes[1:], out[1:]):
        assert rel(o, out[0]) <= 1e-7, mode


def test_fused_sweep_equals_level_sweeps(gpu, monkeypatch):
    """The single-launch solve sweeps (cross-front counters, block tasks for
    every front) and the per-level path with warp-per-front kernels only for
    single-block fronts (RBA_SMALLP=64) agree with the default per-level path
    (warp-per-front kernels up to two pivot blocks) to rounding."""
    prob, _ = rb.build_config("C3", n=8)
    S = mf.analyze(prob.K, prob.dof_coords, 64)
    assert np.any((S["npiv"] > 64) & (S["npiv"] <= 128))   # two-block small fronts exercised
    approx = rb.config_approximant("C3")
    model = prob.true_model()
    outs = []
    for env in ({"RBA_SWEEP": "levels"}, {"RBA_SWEEP": "fused"},
                {"RBA_SWEEP": "levels", "RBA_SMALLP": "64"}):
        for k, val in env.items():
            monkeypatch.setenv(k, val)
        cache = rb.ShiftedFactorCache()
        d = rb.forward_response(prob, model, approx, cache).data
        # single-pole solves advance one slot's sweep counters only; later
        # all-pole sweeps must not wait on the others (per-slot epochs)
        for _ in range(2):
            cache.solve(0, prob.f.astype(complex))
        opr = rb.JacobianOperator(prob, model, approx, cache)
        v = np.random.default_rng(1).standard_normal(opr.shape[1])
        w = np.random.default_rng(2).standard_normal(opr.shape[0])
        outs.append((d, opr.jvp(v), opr.vjp(w)))
        cache.engine.close()
        monkeypatch.delenv("RBA_SMALLP", raising=False)
    # data to 1e-10, J v / J^T w to the parity tolerance 1e-8 (air cells make
    # the adjoint fields ill-conditioned)
    for o in outs[1:]:
        assert rel(outs[0][0], o[0]) <= 1e-10
        assert rel(outs[0][1], o[1]) <= 1e-8
        assert rel(outs[0][2], o[2]) <= 1e-8


def test_blocked_diag_matches_unblocked(gpu, monkeypatch):
    """Both diagonal-block kernels (k_diag: one barrier pair per pivot; k_diag2:
    16x16 sub-blocks) yield the host emulation's factor front by front."""
    prob, _ = rb.build_config("C1", n=10)
    approx = rb.config_approximant("C1")
    model = prob.true_model()
    S = mf.analyze(prob.K, prob.dof_coords, 64)
    A = (prob.K.astype(complex) - approx.poles[1] * orc.assemble_M(prob, model.m)).tocsr()
    panels = mf.factor(A, S)
    outs = []
    for mode in ("v1", "v2"):
        monkeypatch.setenv("RBA_DIAG", mode)
        cache = rb.ShiftedFactorCache()
        rb.factorize_all_poles(prob, model, approx, cache)
        eng = cache.engine
        tot = int(S["panel_off"][-1])
        buf = np.empty(tot, dtype=np.complex128)
        _lib.check(eng.lib.rba_get_factor(eng.ctx, 1, ptr(buf.view(np.float64)), tot))
        outs.append(buf)
        eng.close()
        assert _worst_front_error(buf, panels, S) <= 1e-10, mode
    assert rel(outs[1], outs[0]) <= 1e-7


def test_receiver_green_matches_sweeps(gpu, monkeypatch):
    """J v / J^T w through the receiver Green's functions Z_i = A_i^{-1} Q^T
    (default) equal the per-action triangular sweeps (RBA_GREEN=0) to
    rounding, and the logical solve counters are unchanged."""
    prob, _ = rb.build_config("C3", n=8)
    approx = rb.config_approximant("C3")
    model = prob.true_model()
    outs, counts = [], []
    for green in ("1", "0"):
        monkeypatch.setenv("RBA_GREEN", green)
        cache = rb.ShiftedFactorCache()
        opr = rb.JacobianOperator(prob, model, approx, cache)
        assert opr.engine.info()["green"] == (green == "1")
        v = np.random.default_rng(1).standard_normal(opr.shape[1])
        w = np.random.default_rng(2).standard_normal(opr.shape[0])
        outs.append((opr.jvp(v), opr.vjp(w), opr.jvp(2 * v)))
        counts.append(cache.counters.snapshot())
        if green == "1":
            assert opr.engine.info()["green_builds"] == len(opr.engine.local)
        cache.engine.close()
    assert counts[0] == counts[1]
    for a, b in zip(outs[0], outs[1]):
        assert rel(a, b) <= 1e-9
