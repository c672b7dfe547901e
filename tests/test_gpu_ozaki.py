"""The Ozaki-scheme Schur update on the INT8 tensor cores (kernels_ozaki.cu,
RBA_OZAKI=1): front-by-front against the host emulation of the multifrontal
algorithm, backward error against SuperLU on the C4 shape with 1e-8 S/m air,
and the reference goldens (forward <= 1e-9, J v / J^T w <= 1e-8)."""

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from conftest import golden, rel
import mf_emulator as mf
import paper_2605_19951_b200 as rb
from paper_2605_19951_b200 import _lib
from paper_2605_19951_b200._lib import ptr
from paper_2605_19951_b200.engine import Engine
from oracle import rbainv_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture
def ozaki(monkeypatch):
    monkeypatch.setenv("RBA_OZAKI", "1")
    monkeypatch.setenv("RBA_OZ_MINK", "16")     # small test fronts take the INT8 path too


def _bwd(A, x, b):
    nA = abs(A).sum(axis=1).max()
    return float(np.linalg.norm(A @ x - b) / (nA * np.linalg.norm(x) + np.linalg.norm(b)))


def _front_errors(prob, approx, model):
    cache = rb.ShiftedFactorCache()
    rb.factorize_all_poles(prob, model, approx, cache)
    eng = cache.engine
    S = mf.analyze(prob.K, prob.dof_coords, 64)
    tot = int(S["panel_off"][-1])
    buf = np.empty(tot, dtype=np.complex128)
    out = []
    for pole in (0, 7):
        _lib.check(eng.lib.rba_get_factor(eng.ctx, pole, ptr(buf.view(np.float64)), tot))
        A = (prob.K.astype(complex) - approx.poles[pole] * orc.assemble_M(prob, model.m)).tocsr()
        panels = mf.factor(A, S)
        worst = 0.0
        for s, Lh in enumerate(panels):
            nf, p = S["nf"][s], S["npiv"][s]
            Ld = mf.device_panel_to_ldl(buf[S["panel_off"][s]:S["panel_off"][s] + nf * p]
                                        .reshape(p, nf).T, p)
            mask = np.tril(np.ones((nf, p), bool))
            worst = max(worst, np.abs(Ld[mask] - Lh[mask]).max() / max(np.abs(Lh[mask]).max(), 1e-300))
        out.append(worst)
    eng.close()
    return out


def test_ozaki_fronts_match_emulation(gpu, monkeypatch):
    """Front by front against the host emulation at the C1-shape true model
    (1e-8 S/m air: the entries of the ill-conditioned air fronts differ at the
    1e-10 level between ANY two FP64 orderings).  The INT8 path (Schur and
    aggregated panel updates, every front: RBA_OZ_MINK=16) must stay at the
    level of the all-DMMA factor of the same matrices."""
    prob, _ = rb.build_config("C1", n=10)
    approx = rb.config_approximant("C1")
    model = prob.true_model()
    monkeypatch.setenv("RBA_OZAKI", "0")
    dmma = _front_errors(prob, approx, model)
    monkeypatch.setenv("RBA_OZAKI", "1")
    monkeypatch.setenv("RBA_OZ_MINK", "16")
    monkeypatch.setenv("RBA_OZ_MINROWS", "64")
    oz = _front_errors(prob, approx, model)
    for pole, a, b in zip((0, 7), dmma, oz):
        print(f"fronts pole {pole}: worst front error DMMA {a:.2e}  Ozaki {b:.2e}")
        assert a <= 1e-10
        assert b <= max(1e-10, 3.0 * a)


def test_ozaki_backward_error_c4_shape(gpu, ozaki):
    prob, _ = rb.build_config("C4", n=12)
    approx = rb.config_approximant("C4")
    rng = np.random.default_rng(12)
    b = rng.standard_normal(prob.dof_count) + 1j * rng.standard_normal(prob.dof_count)
    eng = Engine(prob, None)
    eng.set_sources(b[None, :])
    eng.set_poles(approx)
    eng.set_model(prob.m_true)
    eng.factor()
    for i in (0, 5, 10, 15):
        A = (prob.K.astype(complex) - approx.poles[i] *
             orc.assemble_M(prob, prob.m_true).astype(complex)).tocsr()
        e = _bwd(A, eng.solve(i, b), b)
        es = _bwd(A, spla.splu(A.tocsc()).solve(b), b)
        print(f"Ozaki C4-shape pole {i}: backward {e:.2e} (SuperLU {es:.2e})")
        assert e <= max(10 * es, 1e-15)
    eng.close()


def test_ozaki_c1_parity(gpu, ozaki):
    z = golden("ref3d_C1.npz")
    prob, _ = rb.build_config("C1", n=16)
    approx = rb.config_approximant("C1")
    model = rb.Model(z["m"], z["m"])
    cache = rb.ShiftedFactorCache()
    d = rb.forward_response(prob, model, approx, cache).data
    opr = rb.JacobianOperator(prob, model, approx, cache)
    ef, ej, et = rel(d, z["d"]), rel(opr.jvp(z["v"]), z["jv"]), rel(opr.vjp(z["w"]), z["jtw"])
    print(f"Ozaki C1: forward {ef:.2e} J v {ej:.2e} J^T w {et:.2e}")
    assert ef <= 1e-9 and ej <= 1e-8 and et <= 1e-8


def _factor_bytes(monkeypatch, n, wide, pair=False, ts=None):
    monkeypatch.setenv("RBA_OZ_WIDE", "1" if wide else "0")
    if ts is not None:
        monkeypatch.setenv("RBA_OZ_TS", "1" if ts else "0")
    monkeypatch.setenv("RBA_OZ_2CTA", "1" if pair else "0")
    prob, _ = rb.build_config("C4", n=n)
    approx = rb.config_approximant("C4")
    eng = Engine(prob, None)
    eng.set_poles(approx)
    eng.set_model(prob.m_true)
    eng.factor()
    S = mf.analyze(prob.K, prob.dof_coords, 64)
    tot = int(S["panel_off"][-1])
    out = []
    for pole in (0, 9):
        buf = np.empty(tot, dtype=np.complex128)
        _lib.check(eng.lib.rba_get_factor(eng.ctx, pole, ptr(buf.view(np.float64)), tot))
        out.append(buf)
    eng.close()
    return out


def test_ozaki_wide_mma_bitwise(gpu, ozaki, monkeypatch):
    """The default GEMM issues each A digit against runs of up to 4 consecutive
    B digits as ONE MMA of N = 64..256 (10 MMAs per k step); RBA_OZ_WIDE=0
    issues the 28 digit pairs one by one (N = 64).  Same exact int32 sums:
    factors bitwise equal (odd and even row-tile counts, fronts wider than
    one 12-tile super-block)."""
    for n in (10, 20):
        a = _factor_bytes(monkeypatch, n, False)
        b = _factor_bytes(monkeypatch, n, True)
        for x, y in zip(a, b):
            assert np.array_equal(x.view(np.uint64), y.view(np.uint64))


def test_ozaki_cluster_pair_bitwise(gpu, ozaki, monkeypatch):
    """The cluster-pair GEMM (RBA_OZ_2CTA=1: tcgen05.mma.cta_group::2, M = 256,
    each CTA streams its half of every MMA's B rows) sums the same exact int32
    products: factors bitwise equal to the one-SM kernel (odd and even
    row-tile counts, fronts wider than one super-block)."""
    for n in (10, 20):
        a = _factor_bytes(monkeypatch, n, True, False)
        b = _factor_bytes(monkeypatch, n, True, True)
        for x, y in zip(a, b):
            assert np.array_equal(x.view(np.uint64), y.view(np.uint64))


def test_ozaki_ring_depth_and_passes(gpu, ozaki, monkeypatch):
    """RBA_OZ_STAGES=5 (deeper load ring) gives the same bits; RBA_OZ_KMAX=128
    (Schur updates in passes of <= 128 pivots, each with its own row scaling)
    rounds differently but keeps SuperLU's backward error."""
    a = _factor_bytes(monkeypatch, 10, True)
    monkeypatch.setenv("RBA_OZ_STAGES", "5")
    b = _factor_bytes(monkeypatch, 10, True)
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))
    monkeypatch.setenv("RBA_OZ_KMAX", "128")
    prob, _ = rb.build_config("C4", n=10)
    approx = rb.config_approximant("C4")
    eng = Engine(prob, approx)
    eng.set_model(prob.m_true)
    eng.factor()
    M = orc.assemble_M(prob, prob.m_true)
    rng = np.random.default_rng(5)
    rhs = rng.standard_normal(eng.N) + 1j * rng.standard_normal(eng.N)
    for i in (0, 9):
        A = (prob.K.astype(complex) - approx.poles[i] * M.astype(complex)).tocsr()
        e = _bwd(A, eng.solve(i, rhs), rhs)
        print(f"RBA_OZ_KMAX=128 pole {i}: backward error {e:.2e}")
        assert e <= 1e-15
    eng.close()


def test_two_lane_factorisation_bitwise(gpu, ozaki, monkeypatch):
    """RBA_FACTOR_STREAMS=2: the two halves of a pole batch run the plan on two
    streams (own Ozaki digit buffers and tile tickets).  Every pole's factor is
    computed by the same kernels in the same order: bitwise equal."""
    a = _factor_bytes(monkeypatch, 10, True)
    monkeypatch.setenv("RBA_FACTOR_STREAMS", "2")
    b = _factor_bytes(monkeypatch, 10, True)
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))


def test_ozaki_role_counters(gpu, ozaki):
    """rba_oz_prof: the GEMM's own cycle counters are consistent -- k steps and
    tiles counted, waits inside the issuer loop, an SM clock in the B200's
    range (measured with %globaltimer against clock64 inside the kernel)."""
    prob, _ = rb.build_config("C4", n=12)
    approx = rb.config_approximant("C4")
    eng = Engine(prob, approx)
    eng.set_model(prob.m_true)
    eng.oz_prof(True)
    eng.factor()
    pr = eng.oz_prof(True)
    assert pr["tiles"] > 0 and pr["ksteps"] >= pr["tiles"]
    assert 0 <= pr["mma_wait_data"] + pr["mma_wait_tmem"] <= pr["mma_loop"]
    mhz = 1e3 * pr["mma_loop"] / pr["mma_loop_ns"]
    print(f"Ozaki GEMM: {pr['tiles']:.0f} tiles, {pr['ksteps']:.0f} k steps, SM clock {mhz:.0f} MHz")
    assert 500 <= mhz <= 2500
    again = eng.oz_prof(False)
    assert again["tiles"] == 0          # reset by the previous read
    eng.close()


def test_ozaki_tmem_a_bitwise(gpu, ozaki, monkeypatch):
    """RBA_OZ_TS: the A digits staged in TMEM by tcgen05.cp (8 rotating slots
    beside the level accumulators), wide MMAs with A from TMEM -- the same
    exact int32 sums as with A from shared memory: factors bitwise equal."""
    for n in (10, 20):
        a = _factor_bytes(monkeypatch, n, True, False, ts=False)
        b = _factor_bytes(monkeypatch, n, True, False, ts=True)
        for x, y in zip(a, b):
            assert np.array_equal(x.view(np.uint64), y.view(np.uint64))
