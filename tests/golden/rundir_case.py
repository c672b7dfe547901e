"""Deterministic inversion state for the run-directory format pin (shared by
make_golden.py, which writes it with the reference, and tests/test_rundir.py)."""

import numpy as np


def rundir_case():
    """Deterministic single-source inversion state + data for the rundir format."""
    rng = np.random.default_rng(21)
    K_t, M_r, P = 3, 4, 5
    hist = []
    for nu in range(1, 4):
        hist.append(dict(nu=nu, phi=float(rng.random()), misfit=float(rng.random()),
                         reg_value=float(rng.random()), chi2=float(rng.random()),
                         lam=0.5 ** nu, eta=1.0, accepted=bool(nu % 2), lsqr_iters=10 + nu,
                         lsqr_istop=7, wall_ms=100.0 + nu, factorizations=8 * nu,
                         solves=40 * nu, phi_evals=nu, phi_before=float(rng.random()),
                         directional_slope=-float(rng.random())))
    return dict(m=rng.standard_normal(P), m_ref=np.zeros(P), lam=0.125, phi=0.5, chi2=1.25,
                nu=3, diagnostic="max Gauss-Newton iterations",
                counters={"factorizations": 24, "solves": 120}, history=hist,
                d_obs=rng.standard_normal(K_t * M_r), sigma=rng.random(K_t * M_r) + 0.5,
                d_pred=rng.standard_normal(K_t * M_r), times=np.geomspace(1e-5, 1e-3, K_t),
                K_t=K_t, M_r=M_r)
