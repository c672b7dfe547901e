"""Drop-in for rbainv.forward (/root/reference/pkg/src/rbainv/forward.py:32-75).

``forward_response`` solves every pole at the current model on the device
(one multi-RHS sweep per pole for S sources) and combines Q g_i with the
residues in ascending pole order on the device (K10).  The dense
eigen-oracle and implicit-Euler integrators (forward.py:78-127) are
verification tools, out of scope for the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .shifted import ShiftedFactorCache, PoleWorkerPool, SolveError, eng_fields

__all__ = ["ForwardResult", "forward_response", "response_from_pole_solutions"]


@dataclass
class ForwardResult:
    data: np.ndarray                 # (S * K_t * M_r,) [source][channel][receiver]
    fields: np.ndarray | None        # (K_t, N) when retained (S == 1)
    solve_stats: dict


def response_from_pole_solutions(problem, approx, g: np.ndarray, retain_fields: bool = False):
    """Host combination of given pole solutions (forward.py:46-64); used only
    when a caller hands in its own g.  The device path combines in-kernel."""
    res = np.asarray(approx.residues)
    K_t = res.shape[1]
    if retain_fields:
        U = np.zeros((K_t, problem.dof_count))
        for i in range(res.shape[0]):
            U += 2.0 * np.real(np.outer(res[i], g[i]))
        data = np.concatenate([problem.Q @ U[j] for j in range(K_t)])
        return data, U
    D = np.zeros((K_t, problem.Q.shape[0]))
    for i in range(res.shape[0]):
        D += 2.0 * np.real(np.outer(res[i], problem.Q @ g[i]))
    return D.ravel(), None


def forward_device(problem, model, approx, cache: ShiftedFactorCache):
    """Factorise (if needed) and run the forward pass; returns device data."""
    eng = cache.ensure_factored(problem, model, approx)
    d = eng.forward()
    with cache._lock:
        cache.counters.solves += len(eng.local) if eng.comm.world > 1 else eng.m
    return d


def forward_response(problem, model, approx, cache: ShiftedFactorCache,
                     pool: PoleWorkerPool | None = None, retain_fields: bool = False,
                     check_residuals: bool = False) -> ForwardResult:
    d = forward_device(problem, model, approx, cache).cpu().numpy()
    eng = cache.engine
    fields = None
    if retain_fields or check_residuals:
        g = eng_fields(eng)                                   # (m_local, N, S)
        if check_residuals:
            F = problem.source_matrix() if hasattr(problem, "source_matrix") else \
                np.asarray(problem.f, dtype=float)[None, :]
            for i in range(g.shape[0]):
                A = cache.matrix(eng.local[i])
                for s in range(F.shape[0]):
                    nrm = np.linalg.norm(F[s])
                    if nrm > 0:
                        res = np.linalg.norm(A @ g[i, :, s] - F[s]) / nrm
                        if res > 1e-8:
                            raise SolveError(f"pole {eng.local[i]}: relative residual "
                                             f"{res:.3e} exceeds 1e-8")
        if retain_fields:
            # every pole's field, gathered across ranks in pole order
            gall = eng.gather_fields()[:, 0, :].cpu().numpy() if eng.comm.world > 1 \
                else g[:, :, 0]
            d, fields = response_from_pole_solutions(problem, approx, gall, True)
    return ForwardResult(data=d, fields=fields, solve_stats=cache.counters.snapshot())
