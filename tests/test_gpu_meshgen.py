"""3-D operator generation on the GPU (csrc/mesh_gen.cu)
against the host builder mesh3d.build_box_problem (which produced every
golden): identical numbering, dofs, faces, sources and receivers, K equal to
the last bits of the duplicate sums; the device spectral bound against the
host one."""

import time

import numpy as np
import pytest

import paper_2605_19951_b200 as rb
from paper_2605_19951_b200 import mesh3d

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,n", [("C1", 8), ("C3", 8), ("C4", 12), ("C5", 10)])
def test_gpu_box_matches_host(gpu, name, n):
    ph, _ = rb.build_config(name, n=n)
    pd, _ = rb.build_config(name, n=n, device=True)
    for a, b, what in ((ph.cell_dofs, pd.cell_dofs, "cell_dofs"), (ph.grid.cells, pd.grid.cells, "cells"),
                       (ph.grid.dof_of_node, pd.grid.dof_of_node, "dof_of_edge"),
                       (ph.dof_coords, pd.dof_coords, "dof_coords"),
                       (ph.grid.face_cells, pd.grid.face_cells, "face_cells"),
                       (ph.grid.face_measure, pd.grid.face_measure, "face_measure"),
                       (ph.sources, pd.sources, "sources"), (ph.mass_local, pd.mass_local, "mass_local"),
                       (ph.K.indptr, pd.K.indptr, "K indptr"), (ph.K.indices, pd.K.indices, "K indices")):
        np.testing.assert_array_equal(np.asarray(a), np.asarray(b), err_msg=what)
    assert (ph.Q != pd.Q).nnz == 0
    dk = np.abs(ph.K.data - pd.K.data).max() / np.abs(ph.K.data).max()
    print(f"{name} n={n}: K max relative difference {dk:.1e} "
          f"({int((ph.K.data != pd.K.data).sum())} of {ph.K.nnz} entries not bitwise equal)")
    assert dk <= 1e-15
    sb_h = mesh3d.spectral_bound(ph, ph.m_true)
    sb_d = mesh3d.spectral_bound(ph, ph.m_true, device=True)
    assert abs(sb_d - sb_h) <= 1e-12 * sb_h


def test_gpu_box_c4_time(gpu):
    """BASELINE C4 size: GPU generation (incl. downloads) vs the host builder."""
    t0 = time.perf_counter()
    pd, _ = rb.build_config("C4", device=True)
    t1 = time.perf_counter()
    ph, _ = rb.build_config("C4")
    t2 = time.perf_counter()
    print(f"C4 operators: GPU {t1 - t0:.2f} s, host {t2 - t1:.2f} s")
    np.testing.assert_array_equal(ph.cell_dofs, pd.cell_dofs)
    assert pd.K.nnz == ph.K.nnz == 10650286
