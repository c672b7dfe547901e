"""Drop-in for rbainv.shifted on the B200 (factorisation cache + pole solves).

Mirrors /root/reference/pkg/src/rbainv/shifted.py:
``CacheMissError``/``SolveError`` (:36-41), ``CacheCounters`` (:64-70),
``ShiftedFactorCache`` (:73-122), ``PoleWorkerPool`` (:129-155),
``factorize_all_poles`` (:158-173), ``solve_all_poles`` (:176-199),
``resolve_with_cache`` (:202-206).

The cache holds one device `Engine` (libdrba.so).  Two ways in:

* bound mode -- our ``factorize_all_poles``/``solve_all_poles`` bind the cache
  to (problem, approx) and assemble K - xi_i M(m) on the device;
* generic mode -- the reference's *unmodified* ``factorize_all_poles`` calls
  ``cache.factorize(i, A)`` with an assembled SciPy matrix; its values are
  mapped onto the device pattern and factorised the same way.

Either way each pole is a supernodal complex-symmetric LDL^T on the GPU and
``solve`` runs the device triangular sweeps (trans 'T' == 'N': A is complex
symmetric).
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

__all__ = [
    "CacheMissError", "SolveError", "CacheCounters", "ShiftedFactorCache", "PoleWorkerPool",
    "default_worker_count", "factorize_all_poles", "solve_all_poles", "resolve_with_cache",
]


class CacheMissError(KeyError):
    """No factorization cached for the requested pole and model version."""


class SolveError(RuntimeError):
    """Factorization failed or a solve did not meet the residual bound."""


@dataclass
class CacheCounters:
    factorizations: int = 0
    solves: int = 0

    def snapshot(self) -> dict:
        return {"factorizations": self.factorizations, "solves": self.solves}


class _PatternProblem:
    """Minimal problem view for generic mode: the pattern of an assembled A."""

    def __init__(self, A: sp.spmatrix):
        A = sp.csr_matrix(A)
        self.K = sp.csr_matrix((np.zeros(A.nnz), A.indices, A.indptr), shape=A.shape)
        self.cell_dofs = None
        self.mass_local = None
        self.Q = sp.csr_matrix((0, A.shape[0]))
        self.f = np.zeros(A.shape[0])

    def source_matrix(self):
        return self.f[None, :]


class ShiftedFactorCache:
    """Keyed store of device factorizations of A_i(m), one live model version."""

    def __init__(self, backend: str = "gpu", device: int | None = None, leaf: int = 64,
                 max_poles: int = 32):
        if backend not in ("gpu", "sparse", "dense"):
            raise ValueError("backend must be 'gpu' (aliases: 'sparse', 'dense')")
        self.backend = backend
        self.device = device
        self.leaf = leaf
        self.max_poles = max_poles
        self.counters = CacheCounters()
        self.current_tag: str | None = None
        self.engine = None
        self._bound = None          # (id(problem), id(approx)) in bound mode
        self._valid: set[int] = set()
        self._factored_tag = None
        self._A: dict[int, sp.csr_matrix] = {}
        self._lock = threading.Lock()
        self._generic = False
        self._gmap = None

    # ------------------------------------------------------------ binding
    def bind(self, problem, approx):
        key = (id(problem), id(approx))
        if self._bound == key and self.engine is not None:
            return self.engine
        from .engine import Engine
        if self.engine is not None:
            self.engine.close()
        self.engine = Engine(problem, approx, device=self.device, leaf=self.leaf)
        self._bound = key
        self._generic = False
        self._valid = set()
        self._factored_tag = None
        return self.engine

    def slot(self, i: int) -> int:
        try:
            return self.engine.local.index(i)
        except (ValueError, AttributeError):
            raise CacheMissError(f"no factorization for pole {i}, model {self.current_tag}")

    # ------------------------------------------------- reference surface
    def activate(self, tag: str) -> None:
        if tag != self.current_tag:
            self._valid = set()
            self._A = {}
            self.current_tag = tag

    def has(self, i: int, tag: str | None = None) -> bool:
        return (tag or self.current_tag) == self.current_tag and i in self._valid

    def factorize(self, i: int, A: sp.spmatrix) -> None:
        """Generic mode (shifted.py:98-105): factorise an assembled A."""
        if i in self._valid:
            return
        A = sp.csr_matrix(A)
        if self.engine is None or not self._generic or self.engine.N != A.shape[0]:
            from .engine import Engine
            from .parallel import PoleComm
            if PoleComm.current().world > 1:
                # pole i is slot i here: one process owns every pole
                raise RuntimeError("generic mode (factorize(i, A)) is single-process; "
                                   "use factorize_all_poles / forward_response with G > 1")
            if self.engine is not None:
                self.engine.close()
            # factor storage is allocated per pole on its first factorisation,
            # so max_poles only bounds the slot count, not the memory
            self.engine = Engine(_PatternProblem(A), None, device=self.device, leaf=self.leaf,
                                 n_slots=self.max_poles, lazy_factors=True,
                                 comm=PoleComm(1, 0))
            self._generic = True
            self._bound = None
            rows, cols, _, _ = self.engine.pattern()
            self._gmap = (rows.astype(np.int64), cols.astype(np.int64))
        if i >= self.max_poles:
            raise ValueError(f"generic cache holds at most {self.max_poles} poles")
        vals = _values_on_pattern(A, *self._gmap)
        from ._lib import RbaError
        try:
            self.engine.factor_values(i, vals)
        except SolveError:
            raise
        except RbaError as exc:
            raise SolveError(f"factorization of shifted matrix failed: {exc}") from exc
        with self._lock:
            self._valid.add(i)
            self._A[i] = A
            self.counters.factorizations += 1

    def solve(self, i: int, rhs: np.ndarray, trans: str = "N") -> np.ndarray:
        if i not in self._valid:
            raise CacheMissError(f"no factorization for pole {i}, model {self.current_tag}")
        slot = i if self._generic else self.slot(i)
        out = self.engine.solve(slot, np.asarray(rhs, dtype=complex), trans=trans)
        with self._lock:
            self.counters.solves += 1
        return out

    def matrix(self, i: int) -> sp.spmatrix:
        if i not in self._valid:
            raise CacheMissError(f"no factorization for pole {i}, model {self.current_tag}")
        if self._generic:
            return self._A[i]
        if i not in self._A:
            self._A[i] = assembled_matrix(self.engine, self.engine.poles[i])
        return self._A[i]

    # ------------------------------------------------- bound mode helpers
    def ensure_factored(self, problem, model, approx):
        eng = self.bind(problem, approx)
        tag = model.version_tag()
        self.activate(tag)
        owned = set(eng.local)
        if self._factored_tag == tag and owned <= self._valid:
            return eng
        eng.set_model(model.m, tag)
        eng.factor()
        self._factored_tag = tag
        with self._lock:
            self._valid |= owned
            self.counters.factorizations += len(owned)
        return eng


def _values_on_pattern(A: sp.csr_matrix, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """A[rows[e], cols[e]] for the device lower pattern (vectorised lookup)."""
    A = sp.csr_matrix(A)
    A.sum_duplicates()
    n = A.shape[0]
    coo = A.tocoo()
    if coo.nnz == 0:
        return np.zeros(rows.size, dtype=complex)
    keys = coo.row.astype(np.int64) * n + coo.col
    order = np.argsort(keys)
    sk = keys[order]
    want = rows * n + cols
    pos = np.searchsorted(sk, want)
    pos = np.minimum(pos, sk.size - 1)
    hit = sk[pos] == want
    out = np.zeros(rows.size, dtype=complex)
    out[hit] = coo.data[order[pos[hit]]]
    return out


def assembled_matrix(engine, xi: complex) -> sp.csr_matrix:
    """Host copy of A = K - xi M(m) from the device-assembled M (full symmetric)."""
    rows, cols, Kv, Mv = engine.pattern(with_M=True)
    v = Kv - xi * Mv
    off = rows != cols
    r = np.concatenate([rows, cols[off]])
    c = np.concatenate([cols, rows[off]])
    d = np.concatenate([v, v[off]])
    return sp.csr_matrix((d, (r, c)), shape=(engine.N, engine.N))


def default_worker_count() -> int:
    return int(os.environ.get("RBAINV_WORKERS", "1"))


class PoleWorkerPool:
    """Same contract as the reference pool (shifted.py:129-155).  On the GPU the
    poles of one rank are solved together in each launch, so the pool is only
    used for host-side per-pole work; results are pole-indexed."""

    def __init__(self, workers: int = 1):
        self.workers = max(1, int(workers))

    def map_poles(self, fn, count: int) -> list:
        results = [None] * count
        for p in range(self.workers):
            for i in range(p, count, self.workers):
                results[i] = fn(i)
        return results


def factorize_all_poles(problem, model, approx, cache: ShiftedFactorCache,
                        pool: PoleWorkerPool | None = None) -> None:
    """Ensure every A_i = K - xi_i M(m) is factorized for the current model."""
    cache.ensure_factored(problem, model, approx)


def _is_source(problem, rhs) -> bool:
    F = problem.source_matrix() if hasattr(problem, "source_matrix") else \
        np.asarray(problem.f, dtype=float)[None, :]
    return F.shape[0] == 1 and rhs.ndim == 1 and np.array_equal(rhs, F[0])


def solve_all_poles(problem, model, approx, rhs, cache: ShiftedFactorCache,
                    pool: PoleWorkerPool | None = None,
                    check_residuals: bool = False) -> np.ndarray:
    """Solve A_i g_i = rhs for every pole; returns (m, N) complex array."""
    eng = cache.ensure_factored(problem, model, approx)
    rhs = np.asarray(rhs)
    m = approx.pole_count if hasattr(approx, "pole_count") else len(approx.poles)
    if _is_source(problem, rhs):
        eng.forward()
        g = eng.gather_fields()[:, 0, :].cpu().numpy()             # (m, N), all ranks
    elif eng.comm.world == 1:
        g = np.array([eng.solve(cache.slot(i), rhs) for i in range(m)])
    else:
        # each rank solves its own poles; the fields are all-gathered (rank
        # major) and put back in pole order, as PoleWorkerPool's gather
        # (shifted.py:140-155)
        import torch
        nmax = eng.comm.n_max(m)
        loc = torch.zeros((nmax, eng.N), dtype=torch.complex128, device=eng.device)
        rhs_d = torch.as_tensor(np.asarray(rhs, dtype=complex), device=eng.device)
        for slot, i in enumerate(eng.local):
            loc[slot] = eng.solve_d(slot, rhs_d)
        allg = eng._gather(loc)
        idx = torch.as_tensor(eng.slot_of_pole.astype(np.int64), device=eng.device)
        g = allg.index_select(0, idx).cpu().numpy()
    with cache._lock:
        cache.counters.solves += m
    if check_residuals:
        nrm = np.linalg.norm(rhs)
        if nrm > 0:
            for i in range(m):
                res = np.linalg.norm(cache.matrix(i) @ g[i] - rhs) / nrm
                if res > 1e-8:
                    raise SolveError(f"pole {i}: relative residual {res:.3e} exceeds 1e-8")
    return g


def eng_fields(eng) -> np.ndarray:
    """Download the LOCAL g_i (m_local, N, S) in the original dof order."""
    out = []
    for slot in range(len(eng.local)):
        out.append(eng.download_g(slot))
    return np.array(out)


def resolve_with_cache(cache: ShiftedFactorCache, i: int, rhs: np.ndarray,
                       trans: str = "N") -> np.ndarray:
    return cache.solve(i, rhs, trans=trans)
