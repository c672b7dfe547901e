"""NumPy emulation of the device multifrontal algorithm on the host symbolic
structure (test infrastructure).  Mirrors kernels_factor.cu / kernels_solve.cu
step for step: A scattered into the front panels, extend-add of child update
blocks through relmap, pivot-free partial LDL^T, multifrontal forward sweep
with child u-vectors, backward sweep with ancestor gathers."""

import ctypes as C

import numpy as np
import scipy.sparse as sp

from paper_2605_19951_b200 import _lib
from paper_2605_19951_b200._lib import ptr

NAMES32 = ("perm", "first", "npiv", "nf", "parent", "level", "rows", "relmap")
NAMES64 = ("rows_off", "rel_off", "panel_off", "upd_off")


def analyze(A_pattern: sp.csr_matrix, coords=None, leaf=64):
    lib = _lib.load()
    A = sp.csr_matrix(A_pattern)
    A.sort_indices()
    ip = np.ascontiguousarray(A.indptr, dtype=np.int64)
    ix = np.ascontiguousarray(A.indices, dtype=np.int32)
    co = None if coords is None else np.ascontiguousarray(coords, dtype=np.float64)
    h = _lib.vp()
    _lib.check(lib.rba_symbolic_analyze(A.shape[0], ptr(ip), ptr(ix), ptr(co), leaf, C.byref(h)))
    out = {}
    for name in NAMES32 + NAMES64:
        nb = _lib.i64()
        _lib.check(lib.rba_symbolic_array(h, name.encode(), None, 0, C.byref(nb)))
        arr = np.empty(nb.value // (4 if name in NAMES32 else 8),
                       dtype=np.int32 if name in NAMES32 else np.int64)
        _lib.check(lib.rba_symbolic_array(h, name.encode(), ptr(arr), nb.value, C.byref(nb)))
        out[name] = arr
    st = np.zeros(16, np.int64)
    ds = np.zeros(4)
    lib.rba_symbolic_stats(h, ptr(st), ptr(ds))
    out["stats"] = st
    out["flops"] = ds[0]
    lib.rba_symbolic_destroy(h)
    return out


def factor(A: sp.spmatrix, S):
    """Returns per-front dense panels (nf x p) with L below / D on the diagonal."""
    perm = S["perm"]
    Ap = sp.csr_matrix(A)[perm][:, perm].tocsc()
    nfront = S["first"].size
    panels, upd = [], {}
    children = [[] for _ in range(nfront)]
    for c in range(nfront):
        if S["parent"][c] >= 0:
            children[S["parent"][c]].append(c)
    for s in range(nfront):
        f0, p, nf = S["first"][s], S["npiv"][s], S["nf"][s]
        rows = S["rows"][S["rows_off"][s]:S["rows_off"][s + 1]]
        F = np.zeros((nf, nf), dtype=complex)
        blk = Ap[rows][:, f0:f0 + p].toarray()
        F[:, :p] = np.tril(blk)
        for c in children[s]:
            rel = S["relmap"][S["rel_off"][c]:S["rel_off"][c + 1]]
            U = upd.pop(c)
            F[np.ix_(rel, rel)] += np.tril(U)
        for j in range(p):
            d = F[j, j]
            if d == 0 or not np.isfinite(d):
                raise ZeroDivisionError(f"pivot {j} of front {s}")
            w = F[j + 1:, j].copy()
            F[j + 1:, j + 1:] -= np.tril(np.outer(w, w / d))
            F[j + 1:, j] = w / d
        panels.append(F[:, :p].copy())
        if nf > p:
            upd[s] = F[p:, p:].copy()
    return panels


def solve(b: np.ndarray, panels, S):
    perm = S["perm"]
    nfront = S["first"].size
    x = np.asarray(b, dtype=complex)[perm].copy()
    uvec = {}
    children = [[] for _ in range(nfront)]
    for c in range(nfront):
        if S["parent"][c] >= 0:
            children[S["parent"][c]].append(c)
    for s in range(nfront):                          # forward (postorder)
        f0, p, nf = S["first"][s], S["npiv"][s], S["nf"][s]
        L = panels[s]
        v = np.zeros(nf, dtype=complex)
        v[:p] = x[f0:f0 + p]
        for c in children[s]:
            rel = S["relmap"][S["rel_off"][c]:S["rel_off"][c + 1]]
            v[rel] += uvec.pop(c)
        L11 = np.tril(L[:p, :p], -1) + np.eye(p)
        y = np.linalg.solve(L11, v[:p])
        x[f0:f0 + p] = y
        if nf > p:
            uvec[s] = v[p:] - L[p:, :] @ y
    for s in range(nfront - 1, -1, -1):              # backward (reverse postorder)
        f0, p, nf = S["first"][s], S["npiv"][s], S["nf"][s]
        L = panels[s]
        rows = S["rows"][S["rows_off"][s]:S["rows_off"][s + 1]]
        z = x[f0:f0 + p] / np.diag(L[:p, :p])
        if nf > p:
            z = z - L[p:, :].T @ x[rows[p:]]
        L11 = np.tril(L[:p, :p], -1) + np.eye(p)
        x[f0:f0 + p] = np.linalg.solve(L11.T, z)
    out = np.empty_like(x)
    out[perm] = x
    return out


def device_panel_to_ldl(Ld: np.ndarray, p: int, pb: int = 64) -> np.ndarray:
    """Device factor format (fronts.cuh: L' = L D^{1/2} below each 64-pivot
    diagonal block, s = sqrt(d) on the diagonal, unit L inside the diagonal
    blocks) -> the emulator's L (unit lower) / D (diagonal) panel."""
    out = Ld.copy()
    for j in range(p):
        s = Ld[j, j]
        b1 = min((j // pb + 1) * pb, p)
        out[b1:, j] = Ld[b1:, j] / s
        out[j, j] = s * s
    return out
