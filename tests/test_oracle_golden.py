"""The CPU oracle (oracle/rbainv_oracle.py) is pinned against golden vectors
produced by the unmodified reference (tests/golden/make_golden.py)."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden, rel
from oracle import rbainv_oracle as orc
import paper_2605_19951_b200 as rb


class _P:
    """Problem view rebuilt from the golden arrays (2-D reference fixture)."""

    def __init__(self, z):
        N = z["K_indptr"].size - 1
        self.K = sp.csr_matrix((z["K_data"], z["K_indices"], z["K_indptr"]), shape=(N, N))
        self.Q = sp.csr_matrix((z["Q_data"], z["Q_indices"], z["Q_indptr"]),
                               shape=tuple(z["Q_shape"]))
        self.cell_dofs = z["cell_dofs"]
        self.mass_local = z["mass_local"]
        self.f = z["f"]
        self.sources = None
        self._scatter = None


def test_oracle_matches_reference_2d():
    z = golden("ref2d_small.npz")
    p = _P(z)
    fac = orc.PoleFactors()
    d, g = orc.forward_response(p, z["m"], z["poles"], z["residues"], fac)
    assert rel(g[:, :, 0], z["g"][:, :, 0]) <= 1e-14
    assert rel(d, z["d"]) <= 1e-14
    J = orc.Jacobian(p, z["m"], z["poles"], z["residues"], fac, g=g)
    assert rel(J.jvp(z["v"]), z["jv"]) <= 1e-13
    assert rel(J.vjp(z["w"]), z["jtw"]) <= 1e-13
    R = sp.csr_matrix(z["R_dense"])
    for k in (1, 3, 5):
        dm, itn, _ = orc.augmented_lsqr(J, R, 1.0 / z["sigma_d"], z["d_obs"], d, z["m"],
                                        z["m_ref"], float(z["lam"]), 0.0, k)
        assert itn == int(z[f"itn_{k}"])
        assert rel(dm, z[f"dm_{k}"]) <= 1e-9


@pytest.mark.parametrize("fname,name", [("ref3d_n6.npz", "C1"), ("ref3d_c3_n6.npz", "C3")])
def test_oracle_matches_reference_3d(fname, name):
    z = golden(fname)
    prob, meta = rb.build_config(name, n=int(z["n"]))
    # the golden run stored the problem arrays: the 3-D builder is deterministic
    assert np.array_equal(prob.cell_dofs, z["cell_dofs"])
    assert np.allclose(prob.mass_local, z["mass_local"], rtol=0, atol=0)
    approx = rb.config_approximant(name)
    fac = orc.PoleFactors()
    d, g = orc.forward_response(prob, z["m"], approx.poles, approx.residues, fac)
    assert rel(d, z["d"]) <= 1e-13
    J = orc.Jacobian(prob, z["m"], approx.poles, approx.residues, fac, g=g)
    assert rel(J.jvp(z["v"]), z["jv"]) <= 1e-12
    assert rel(J.vjp(z["w"]), z["jtw"]) <= 1e-12
    reg = orc.build_reg(prob.grid)
    dm, itn, _ = orc.augmented_lsqr(J, reg["R"], 1.0 / z["sigma_d"], z["d_obs"], d, z["m"],
                                    z["m"], float(z["lam"]), 0.0, 1)
    assert rel(dm, z["dm_1"]) <= 1e-9


def test_face_root_squares_to_L():
    prob, _ = rb.build_config("C1", n=4)
    reg = orc.build_reg(prob.grid, dense_chol=False)
    Rt = orc.face_root(reg, prob.grid)
    diff = (Rt.T @ Rt - reg["L"]).toarray()
    assert np.abs(diff).max() <= 1e-12 * np.abs(reg["L"].toarray()).max()


def test_golden_c1_present_and_consistent():
    z = golden("ref3d_C1.npz")
    assert int(z["n"]) == 16
    assert z["d"].size == 31 * 20
    assert z["jtw"].size == 6 * 16 ** 3
    # the reference's own adjointness on C1 (SURVEY §0.9 measured 3-4e-9 on its probe)
    assert float(z["adjoint"]) < 1e-7
