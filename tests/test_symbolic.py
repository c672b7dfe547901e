"""Host symbolic analysis (libdrba.so, no GPU): structure invariants and an
exact NumPy emulation of the device multifrontal factor/solve on it."""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from conftest import rel
import mf_emulator as mf
import paper_2605_19951_b200 as rb
from oracle import rbainv_oracle as orc


def _shifted(prob, m, xi):
    M = orc.assemble_M(prob, m)
    return (prob.K.astype(complex) - xi * M.astype(complex)).tocsr()


@pytest.mark.parametrize("n,leaf,geo", [(4, 16, True), (6, 64, True), (6, 32, False), (8, 64, True)])
def test_structure_invariants(n, leaf, geo):
    prob, _ = rb.build_config("C1", n=n)
    S = mf.analyze(prob.K, prob.dof_coords if geo else None, leaf)
    N = prob.dof_count
    perm = S["perm"]
    assert np.array_equal(np.sort(perm), np.arange(N))
    first, npiv, nf, parent = S["first"], S["npiv"], S["nf"], S["parent"]
    # fronts partition the permuted index space, children before parents
    assert np.array_equal(np.cumsum(npiv)[:-1], first[1:])
    assert all(parent[s] == -1 or parent[s] > s for s in range(first.size))
    Ap = sp.csr_matrix(prob.K)[perm][:, perm].tocoo()
    # every lower entry of A lies inside the front that owns its column
    owner = np.repeat(np.arange(first.size), npiv)
    for r, c in zip(Ap.row, Ap.col):
        if r < c:
            continue
        s = owner[c]
        rows = S["rows"][S["rows_off"][s]:S["rows_off"][s + 1]]
        assert r in rows
    # a child's border is contained in its parent's rows
    for c in range(first.size):
        p = parent[c]
        if p < 0:
            assert nf[c] == npiv[c]
            continue
        crow = S["rows"][S["rows_off"][c] + npiv[c]:S["rows_off"][c + 1]]
        prow = S["rows"][S["rows_off"][p]:S["rows_off"][p + 1]]
        rel_ = S["relmap"][S["rel_off"][c]:S["rel_off"][c + 1]]
        assert np.array_equal(prow[rel_], crow)


@pytest.mark.parametrize("n,leaf", [(4, 16), (6, 64)])
def test_emulated_multifrontal_solve(n, leaf):
    prob, _ = rb.build_config("C1", n=n)
    m = prob.m_true
    approx = rb.config_approximant("C1")
    S = mf.analyze(prob.K, prob.dof_coords, leaf)
    rng = np.random.default_rng(0)
    b = rng.standard_normal(prob.dof_count) + 1j * rng.standard_normal(prob.dof_count)
    for xi in approx.poles[:3]:
        A = _shifted(prob, m, xi)
        panels = mf.factor(A, S)
        x = mf.solve(b, panels, S)
        ref = spla.splu(A.tocsc()).solve(b)
        r = np.linalg.norm(A @ x - b)
        # reference criterion (shifted.py:193-196) and normwise backward error
        assert r / np.linalg.norm(b) <= 1e-8
        assert r / (abs(A).sum(axis=1).max() * np.linalg.norm(x) + np.linalg.norm(b)) <= 1e-15
        assert rel(x, ref) <= 1e-8


def test_flop_and_fill_stats_c1():
    prob, _ = rb.build_config("C1", n=16)
    S = mf.analyze(prob.K, prob.dof_coords, 64)
    st = S["stats"]
    # SURVEY §0.10 measured geometric-ND fill 5.74e6 / 1.05e10 flops, max column 1,096
    assert 5.0e6 < st[3] < 7.5e6
    assert 0.8e10 < S["flops"] < 1.4e10
    assert st[7] == 1096


@pytest.mark.parametrize("name,n", [("C1", 6), ("C3", 6)])
def test_mesh_prepare_dry_run(name, n):
    """rba_set_mesh's host preparation (pattern, symbolic, scatter plan) runs
    without a GPU; every lower entry of A must land in a front panel."""
    from paper_2605_19951_b200 import _lib
    from paper_2605_19951_b200._lib import ptr
    lib = _lib.load()
    prob, _ = rb.build_config(name, n=n)
    K = sp.csr_matrix(prob.K)
    K.sort_indices()
    cd = np.ascontiguousarray(prob.cell_dofs, dtype=np.int32)
    ml = np.ascontiguousarray(prob.mass_local)
    kp = np.ascontiguousarray(K.indptr, dtype=np.int64)
    ki = np.ascontiguousarray(K.indices, dtype=np.int32)
    kx = np.ascontiguousarray(K.data)
    co = np.ascontiguousarray(prob.dof_coords)
    out = np.zeros(4, np.int64)
    _lib.check(lib.rba_mesh_prepare(K.shape[0], prob.grid.cell_count, 6, ptr(cd), ptr(ml),
                                    ptr(kp), ptr(ki), ptr(kx), ptr(co), 64, ptr(out)))
    assert out[0] == (K.nnz + K.shape[0]) // 2
    # every cell contributes its 21 lower (a, b) pairs with both dofs interior
    assert out[1] == sum(int(((r >= 0)[:, None] & (r >= 0)[None, :] &
                              (r[:, None] >= r[None, :])).sum()) for r in prob.cell_dofs)
