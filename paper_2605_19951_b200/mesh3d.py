"""3-D lowest-order Nedelec (Whitney edge) problems on Kuhn-split hex boxes.

The reference builds only 1-D/2-D P1 grids (mesh.py:294-306).
This module is the host-side 3-D restatement that SURVEY.md §8c asks for:
it emits a `Problem` with exactly the reference's algebraic roles

* ``K``            curl-curl stiffness (1/mu) int curl N_a . curl N_b   (CSR, N x N)
* ``mass_local``   unit-conductivity local mass int N_a . N_b, edge signs folded in
* ``cell_dofs``    (P, 6) dof per local edge, -1 on PEC (tangential-E = 0) edges,
                   mirroring the Dirichlet elimination of mesh.py:233-239
* ``f``/``sources`` loop currents: f_e = +-I on the edges the loop runs along
* ``Q``            -z . curl E at receivers (dB_z/dt up to sign), constant per tet
* ``grid``         cell measures and interior-face adjacency for RT0 regularisation

so the reference's own ``assemble_M`` / ``dM_contract`` / solves / Jacobian /
LSQR run on it unchanged.  Everything is vectorised numpy (n=64 has 1.57M tets).

Geometry: unit-spaced vertices (i, j, k) * h, z up; every hex is split into the
6 Kuhn tets v0 -> v0+e_a -> v0+e_a+e_b -> v0+(1,1,1) (one per axis permutation),
which is conforming across hexes.  Vertex ids grow along every axis, so each
tet's vertices are already in increasing global order and every local edge is
oriented low -> high (all orientation signs are +1; the sign code stays general).
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .problem import Grid, Problem

__all__ = ["BoxSpec", "build_box_problem", "LOCAL_EDGES", "MU0", "kuhn_tet_of_point",
           "config_spec", "build_config", "spectral_bound"]

MU0 = 4e-7 * np.pi
LOCAL_EDGES = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))
_PERMS = tuple(itertools.permutations(range(3)))


@dataclass(frozen=True)
class BoxSpec:
    n: int                               # hexes per axis
    n_air: int = 4                       # top hex layers that are air
    h: float = 1.0                       # hex edge length
    mu: float = MU0
    sigma_background: float = 0.01
    sigma_air: float = 1e-8
    loops: tuple = ()                    # ((x0, y0, size), ...) at the air/ground interface
    receivers: tuple = ()                # ((x, y, z), ...) strictly inside tets
    current: float = 1.0


def _vid(n, x, y, z):
    return x + (n + 1) * (y + (n + 1) * z)


def kuhn_tet_of_point(n, p, h=1.0):
    """Tet index containing point p (strictly interior), with the tet
    numbering of `build_box_problem`."""
    q = np.asarray(p, dtype=float) / h
    ijk = np.floor(q).astype(int)
    frac = q - ijk
    if np.any(ijk < 0) or np.any(ijk >= n):
        raise ValueError(f"point {p} outside the box")
    order = tuple(int(a) for a in np.argsort(-frac, kind="stable"))
    if len(set(np.round(frac, 12))) < 3 or np.any(frac <= 0) or np.any(frac >= 1):
        raise ValueError(f"point {p} is not strictly inside a tet")
    hexid = ijk[0] + n * (ijk[1] + n * ijk[2])
    return hexid * 6 + _PERMS.index(order)


def _local_matrices(h, mu):
    """Mass and stiffness of the 6 Kuhn tet shapes (translation invariant)."""
    mass = np.zeros((6, 6, 6))
    stiff = np.zeros((6, 6, 6))
    curls = np.zeros((6, 6, 3))
    vol = h ** 3 / 6.0
    for t, perm in enumerate(_PERMS):
        v = np.zeros((4, 3))
        for s in range(3):
            v[s + 1] = v[s]
            v[s + 1][perm[s]] += h
        T = (v[1:] - v[0]).T                        # columns = edge vectors
        Ginv = np.linalg.inv(T)                     # rows = grad lambda_1..3
        grads = np.vstack([-Ginv.sum(axis=0), Ginv])
        G = grads @ grads.T
        II = vol * (np.ones((4, 4)) + np.eye(4)) / 20.0
        for a, (i, j) in enumerate(LOCAL_EDGES):
            curls[t, a] = 2.0 * np.cross(grads[i], grads[j])
            for b, (k, l) in enumerate(LOCAL_EDGES):
                mass[t, a, b] = (G[j, l] * II[i, k] - G[j, k] * II[i, l]
                                 - G[i, l] * II[j, k] + G[i, k] * II[j, l])
        stiff[t] = vol / mu * curls[t] @ curls[t].T
    return mass, stiff, curls, vol


def _box_topology_host(spec, nodes, tet_type, mass6, stiff6):
    """Host NumPy path of build_box_problem's topology (the reference layout):
    tets, edge numbering (np.unique of (low, high) vertex keys), PEC edges,
    dofs, K (COO -> CSR), edge midpoints, interior faces."""
    n, h = spec.n, spec.h
    NV1 = n + 1
    NVt = nodes.shape[0]
    hx, hy, hz = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    hx, hy, hz = hx.ravel(order="F"), hy.ravel(order="F"), hz.ravel(order="F")
    # hex id = x + n*(y + n*z) ordering (x fastest)
    H = n ** 3
    cells = np.empty((H, 6, 4), dtype=np.int64)
    for t, perm in enumerate(_PERMS):
        cx, cy, cz = hx.copy(), hy.copy(), hz.copy()
        cells[:, t, 0] = _vid(n, cx, cy, cz)
        for s in range(3):
            if perm[s] == 0:
                cx = cx + 1
            elif perm[s] == 1:
                cy = cy + 1
            else:
                cz = cz + 1
            cells[:, t, s + 1] = _vid(n, cx, cy, cz)
    cells = cells.reshape(H * 6, 4)
    P = cells.shape[0]
    la = np.array([e[0] for e in LOCAL_EDGES])
    lb = np.array([e[1] for e in LOCAL_EDGES])
    va, vb = cells[:, la], cells[:, lb]                     # (P, 6)
    lo, hi = np.minimum(va, vb), np.maximum(va, vb)
    sign = np.where(vb > va, 1.0, -1.0)
    keys = lo * NVt + hi
    ukeys, inv = np.unique(keys.ravel(), return_inverse=True)
    cell_edges = inv.reshape(P, 6)
    e_lo, e_hi = ukeys // NVt, ukeys % NVt
    pa, pb = nodes[e_lo] / h, nodes[e_hi] / h
    on_bnd = np.zeros(ukeys.size, dtype=bool)
    for ax in range(3):
        on_bnd |= (pa[:, ax] == 0) & (pb[:, ax] == 0)
        on_bnd |= (pa[:, ax] == n) & (pb[:, ax] == n)
    dof_of_edge = -np.ones(ukeys.size, dtype=np.int64)
    N = int((~on_bnd).sum())
    dof_of_edge[~on_bnd] = np.arange(N)
    cell_dofs = dof_of_edge[cell_edges]
    dof_coords = (0.5 * (nodes[e_lo] + nodes[e_hi]))[~on_bnd]
    S = sign[:, :, None] * sign[:, None, :]
    mass_local = mass6[tet_type] * S
    stiff_local = stiff6[tet_type] * S
    k = 6
    rows = np.repeat(cell_dofs, k, axis=1).ravel()
    cols = np.tile(cell_dofs, (1, k)).ravel()
    keep = (rows >= 0) & (cols >= 0)
    K = sp.coo_matrix((stiff_local.ravel()[keep], (rows[keep], cols[keep])),
                      shape=(N, N)).tocsr()
    # interior faces (RT0 regulariser adjacency)
    fl = np.array([(0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3)])
    tri = np.sort(cells[:, fl], axis=2).reshape(-1, 3)                   # (4P, 3)
    fkeys = (tri[:, 0] * NVt + tri[:, 1]) * NVt + tri[:, 2]
    order = np.argsort(fkeys, kind="stable")
    sk = fkeys[order]
    dup = np.flatnonzero(sk[1:] == sk[:-1])
    owner = np.repeat(np.arange(P), 4)
    face_cells = np.column_stack([owner[order[dup]], owner[order[dup + 1]]])
    t0 = tri[order[dup]]
    p0, p1, p2 = nodes[t0[:, 0]], nodes[t0[:, 1]], nodes[t0[:, 2]]
    face_measure = 0.5 * np.linalg.norm(np.cross(p1 - p0, p2 - p0), axis=1)
    edge_index = {int(kk): i for i, kk in enumerate(ukeys)} if len(spec.loops) else {}

    def dof_of(a, b):
        return int(dof_of_edge[edge_index[int(min(a, b) * NVt + max(a, b))]])
    return (P, N, cells, cell_dofs, K, dof_of_edge, dof_coords, face_cells, face_measure, sign,
            mass_local, stiff_local, dof_of)


_DIRS = ((1, 0, 0), (0, 1, 0), (1, 1, 0), (0, 0, 1), (1, 0, 1), (0, 1, 1), (1, 1, 1))


def _interior_mask(n, x, y, z):
    """Edge directions (bit d: _DIRS[d]) leaving vertex (x, y, z) that exist in
    the box and are not PEC edges (both ends on one boundary plane)."""
    mask = 0
    for d, (dx, dy, dz) in enumerate(_DIRS):
        if x + dx > n or y + dy > n or z + dz > n:
            continue
        bnd = (dx == 0 and x in (0, n)) or (dy == 0 and y in (0, n)) or (dz == 0 and z in (0, n))
        if not bnd:
            mask |= 1 << d
    return mask


def _box_topology_gpu(n, h, stiff6):
    """Edge numbering, tet vertices / dofs, curl-curl K, edge midpoints and the
    interior-face adjacency generated on the GPU (csrc/mesh_gen.cu,
    rba_box_generate) -- the same numbering as the host path below."""
    import ctypes as C
    from . import _lib
    lib = _lib.load()
    h_ = _lib.vp()
    st6 = np.ascontiguousarray(stiff6.reshape(6, 36), dtype=np.float64)
    rc = lib.rba_box_generate(int(n), float(h), st6.ctypes.data, C.byref(h_))
    if rc != 0:
        raise RuntimeError("GPU mesh generation failed: " + lib.rba_box_last_error().decode())
    info = np.zeros(6, np.int64)
    lib.rba_box_info(h_, info.ctypes.data)
    N, P, nnz, F, E, NVt = (int(v) for v in info)

    def get(name, shape, dtype):
        a = np.empty(shape, dtype=dtype)
        rc2 = lib.rba_box_get(h_, name.encode(), a.ctypes.data, a.nbytes)
        if rc2 != 0:
            raise RuntimeError(lib.rba_box_last_error().decode())
        return a
    try:
        out = dict(N=N, P=P,
                   cells=get("cells", (P, 4), np.int64),
                   cell_dofs=get("cell_dofs", (P, 6), np.int32).astype(np.int64),
                   K=sp.csr_matrix((get("data", nnz, np.float64), get("indices", nnz, np.int32),
                                    get("indptr", N + 1, np.int64)), shape=(N, N)),
                   face_cells=get("face_cells", (F, 2), np.int32).astype(np.int64),
                   face_measure=get("face_measure", F, np.float64),
                   dof_of_edge=get("dof_of_edge", E, np.int64),
                   dof_coords=get("dof_coords", (N, 3), np.float64),
                   dof_offset=get("dof_offset", NVt + 1, np.int64))
    finally:
        lib.rba_box_destroy(h_)
    return out


def build_box_problem(spec: BoxSpec, m_true=None, device: bool = False) -> Problem:
    """The 3-D Nedelec `Problem` of a BoxSpec.  device=True generates the
    topology and K on the GPU (rba_box_generate: the same numbering and the
    same element-order duplicate sums); the default is the host NumPy path."""
    n, h = spec.n, spec.h
    NV1 = n + 1
    H = n ** 3
    tet_type = np.tile(np.arange(6), H)
    gx, gy, gz = np.meshgrid(np.arange(NV1), np.arange(NV1), np.arange(NV1), indexing="ij")
    nodes = np.column_stack([gx.ravel(order="F"), gy.ravel(order="F"),
                             gz.ravel(order="F")]).astype(float) * h
    NVt = nodes.shape[0]
    mass6, stiff6, curl6, vol = _local_matrices(h, spec.mu)
    if device:
        g = _box_topology_gpu(n, h, stiff6)
        P, N = g["P"], g["N"]
        cells, cell_dofs, K = g["cells"], g["cell_dofs"], g["K"]
        dof_of_edge, dof_coords = g["dof_of_edge"], g["dof_coords"]
        face_cells, face_measure = g["face_cells"], g["face_measure"]
        sign = np.ones((P, 6))                    # vertex ids increase along every tet edge
        mass_local = mass6[tet_type]
        stiff_local = stiff6[tet_type]
        doff = g["dof_offset"]

        def dof_of(a, b):
            lo, hi = min(a, b), max(a, b)
            x, y, z = lo % NV1, (lo // NV1) % NV1, lo // (NV1 * NV1)
            dx, dy, dz = hi % NV1 - x, (hi // NV1) % NV1 - y, hi // (NV1 * NV1) - z
            d = _DIRS.index((dx, dy, dz))
            mask = _interior_mask(n, x, y, z)
            if not mask >> d & 1:
                return -1
            return int(doff[lo]) + bin(mask & ((1 << d) - 1)).count("1")
    else:
        (P, N, cells, cell_dofs, K, dof_of_edge, dof_coords, face_cells, face_measure, sign,
         mass_local, stiff_local, dof_of) = _box_topology_host(spec, nodes, tet_type, mass6,
                                                              stiff6)
    cell_measure = np.full(P, vol)

    # --- sources: square loops at the air/ground interface ----------------
    z_if = n - spec.n_air
    srcs = []
    for (x0, y0, size) in spec.loops:
        f = np.zeros(N)
        path = [(x0 + i, y0, 0, +1) for i in range(size)]                 # +x along y=y0
        path += [(x0 + size, y0 + i, 1, +1) for i in range(size)]         # +y along x=x0+L
        path += [(x0 + size - 1 - i, y0 + size, 0, -1) for i in range(size)]  # -x
        path += [(x0, y0 + size - 1 - i, 1, -1) for i in range(size)]     # -y
        for (x, y, ax, direction) in path:
            a = _vid(n, x, y, z_if)
            b = _vid(n, x + (ax == 0), y + (ax == 1), z_if)
            d = dof_of(a, b)
            if d < 0:
                raise ValueError("source loop touches the PEC boundary")
            f[d] += spec.current * direction * (1.0 if b > a else -1.0)
        srcs.append(f)
    sources = np.array(srcs) if srcs else np.zeros((1, N))

    # --- receivers: -(curl E)_z in the containing tet ----------------------
    recv = np.atleast_2d(np.asarray(spec.receivers, dtype=float)) if len(spec.receivers) \
        else np.zeros((0, 3))
    q_rows, q_cols, q_vals = [], [], []
    for r, pos in enumerate(recv):
        c = kuhn_tet_of_point(n, pos, h)
        for a in range(6):
            d = cell_dofs[c, a]
            val = -curl6[tet_type[c], a, 2] * sign[c, a]
            if d < 0:
                if val != 0.0:
                    raise ValueError(f"receiver {pos} touches an eliminated PEC edge")
                continue
            if val != 0.0:
                q_rows.append(r)
                q_cols.append(d)
                q_vals.append(val)
    Q = sp.coo_matrix((q_vals, (q_rows, q_cols)), shape=(recv.shape[0], N)).tocsr()

    grid = Grid(dimension=3, nodes=nodes, cells=cells, cell_measure=cell_measure,
                face_cells=face_cells, face_measure=face_measure,
                dof_of_node=dof_of_edge, dof_count=N,
                cell_tags=np.full(P, "", dtype=object))
    prob = Problem(grid=grid, K=K, cell_dofs=cell_dofs, mass_local=mass_local,
                   stiff_local=stiff_local, f=sources[0].copy(), Q=Q, receivers=recv,
                   spec=spec, sources=sources, dof_coords=dof_coords,
                   m_true=None if m_true is None else np.asarray(m_true, dtype=float),
                   sigma_background=spec.sigma_background)
    prob.extra["tet_type"] = tet_type
    prob.extra["z_interface"] = z_if
    return prob


def cell_centroids_box(n, h=1.0):
    """Tet centroids in `build_box_problem` order without building the mesh."""
    hx, hy, hz = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    base = np.column_stack([hx.ravel(order="F"), hy.ravel(order="F"),
                            hz.ravel(order="F")]).astype(float)
    offs = []
    for perm in _PERMS:
        v = np.zeros((4, 3))
        for s in range(3):
            v[s + 1] = v[s]
            v[s + 1][perm[s]] += 1.0
        offs.append(v.mean(axis=0))
    offs = np.array(offs)
    return ((base[:, None, :] + offs[None, :, :]).reshape(-1, 3)) * h


def spectral_bound(problem: Problem, m: np.ndarray, device: bool = False) -> float:
    """Largest generalized eigenvalue over the element pencils
    (stiff_c, e^{m_c} mass_c) -- vectorised form of the reference's
    `spectral_bound` (mesh.py:406-421).  The curl-curl pencil is singular in K
    but M_c is SPD, so Cholesky of M_c is safe.  device=True: one Cholesky +
    power iteration per cell on the GPU (rba_spectral_bound), any mesh."""
    if device:
        from . import _lib
        lib = _lib.load()
        ml = np.ascontiguousarray(problem.mass_local, dtype=np.float64)
        sl = np.ascontiguousarray(problem.stiff_local, dtype=np.float64)
        mm = np.ascontiguousarray(m, dtype=np.float64)
        out = np.zeros(1)
        rc = lib.rba_spectral_bound(ml.shape[0], ml.ctypes.data, sl.ctypes.data, mm.ctypes.data,
                                    out.ctypes.data)
        if rc != 0:
            raise RuntimeError("rba_spectral_bound failed: " + lib.rba_box_last_error().decode())
        return float(out[0])
    tt = problem.extra.get("tet_type")
    if tt is not None:
        best = 0.0
        sig = np.exp(m)
        for t in range(6):
            sel = np.flatnonzero(tt == t)
            if sel.size == 0:
                continue
            c = sel[0]
            Lc = np.linalg.cholesky(problem.mass_local[c])
            Li = np.linalg.inv(Lc)
            w = np.linalg.eigvalsh(Li @ problem.stiff_local[c] @ Li.T)[-1]
            best = max(best, float(w / sig[sel].min()))
        return best
    Lc = np.linalg.cholesky(problem.mass_local * np.exp(m)[:, None, None])
    Li = np.linalg.inv(Lc)
    A = Li @ problem.stiff_local @ np.swapaxes(Li, 1, 2)
    return float(np.linalg.eigvalsh(A)[:, -1].max())


# ---------------------------------------------------------------------------
# BASELINE.json configurations (synthetic stand-ins)
# ---------------------------------------------------------------------------

def _line_receivers(n, z_if, count, y_frac=0.61, z_frac=0.23):
    """`count` points on a line along x at the air side of the interface,
    evenly spread and nudged so every point is strictly inside one tet."""
    xs = np.linspace(1.07, n - 1.07, count)
    fr = xs - np.floor(xs)
    bad = (np.abs(fr - y_frac) < 1e-3) | (np.abs(fr - z_frac) < 1e-3) | (fr < 1e-3)
    xs[bad] += 0.011
    yc = n // 2
    return tuple((float(x), yc + y_frac, z_if + z_frac) for x in xs)


def _grid_receivers(n, z_if, side, x_frac=0.37, y_frac=0.61, z_frac=0.23):
    span = n - 4
    pos = np.linspace(2, 2 + span - 1, side).astype(int)
    return tuple((x + x_frac, y + y_frac, z_if + z_frac) for y in pos for x in pos)


def _loops(n, count, size):
    if count == 1:
        c = (n - size) // 2
        return ((c, c, size),)
    out = []
    step = max(1, (n - 2 - size) // max(1, int(np.ceil(np.sqrt(count))) - 1)) \
        if count > 1 else 0
    side = int(np.ceil(np.sqrt(count)))
    for k in range(count):
        i, j = k % side, k // side
        x0 = 1 + min(i * step, n - 2 - size)
        y0 = 1 + min(j * step, n - 2 - size)
        out.append((x0, y0, size))
    return tuple(out)


def config_spec(name: str, n: int | None = None) -> tuple[BoxSpec, dict]:
    """BoxSpec plus model/inversion metadata for BASELINE configs C1..C5.
    ``n`` overrides the mesh size (tests use small boxes of the same shape)."""
    name = name.upper()
    if name == "C1":
        n = n or 16
        n_air = 4 if n >= 8 else 1
        z_if = n - n_air
        size = min(8, n - 4)
        spec = BoxSpec(n=n, n_air=n_air, sigma_background=0.01,
                       loops=_loops(n, 1, size),
                       receivers=_line_receivers(n, z_if, 20 if n >= 12 else max(2, n - 2)))
        meta = dict(poles=8, times=(1e-5, 1e-2, 31), lsqr_iters=20, lam=1e-2,
                    noise=(0.01, 0), block=4)
    elif name in ("C2", "C3"):
        n = n or 32
        n_air = 4 if n >= 8 else 1
        z_if = n - n_air
        size = min(8, (n - 4) // 2) if name == "C3" else min(8, n - 4)
        spec = BoxSpec(n=n, n_air=n_air, sigma_background=0.01,
                       loops=_loops(n, 1 if name == "C2" else 4, size),
                       receivers=() if name == "C2" else
                       _grid_receivers(n, z_if, min(10, n - 4)))
        meta = dict(poles=16, times=(1e-5, 1e-2, 31), nrhs=4, seed=1, trials=50)
    elif name == "C4":
        n = n or 46
        n_air = 6 if n >= 12 else 1
        z_if = n - n_air
        size = min(8, (n - 4) // 2)
        spec = BoxSpec(n=n, n_air=n_air, sigma_background=0.005,
                       loops=_loops(n, 4, size),
                       receivers=_grid_receivers(n, z_if, min(10, n - 4)))
        meta = dict(poles=16, times=(1e-5, 1e-2, 31), lsqr_iters=30, lam=1e-2,
                    noise=(0.02, 2), gn_iters=10, m0=0.01)
    elif name == "C5":
        n = n or 64
        n_air = 6 if n >= 12 else 1
        z_if = n - n_air
        size = min(8, (n - 4) // 3)
        spec = BoxSpec(n=n, n_air=n_air, sigma_background=0.01,
                       loops=_loops(n, 8, size),
                       receivers=_grid_receivers(n, z_if, min(20, n - 4)))
        meta = dict(poles=20, times=(1e-6, 1e-2, 41), lsqr_iters=30, seed=3)
    else:
        raise ValueError(f"unknown config {name}")
    meta["name"] = name
    meta["n"] = n
    return spec, meta


def config_true_model(name: str, spec: BoxSpec) -> np.ndarray:
    """Per-tet log-conductivity of each config's true model."""
    name = name.upper()
    n = spec.n
    cz = cell_centroids_box(n, spec.h) / spec.h
    z_if = n - spec.n_air
    air = cz[:, 2] > z_if
    sig = np.full(cz.shape[0], spec.sigma_background)
    if name == "C1":
        b = 4 if n >= 12 else max(1, n // 4)
        x0 = (n - b) / 2
        z1 = z_if - 2 if n >= 12 else z_if
        inb = ((cz[:, 0] > x0) & (cz[:, 0] < x0 + b) & (cz[:, 1] > x0) & (cz[:, 1] < x0 + b)
               & (cz[:, 2] > z1 - b) & (cz[:, 2] < z1))
        sig[inb] = 1.0
    elif name == "C2":
        rng = np.random.default_rng(1)
        sig = np.exp(rng.uniform(np.log(1e-3), np.log(1.0), cz.shape[0]))
        air[:] = False
    elif name == "C3":
        b = 6 if n >= 24 else max(1, n // 5)
        z1 = z_if - 2
        for x0, s in ((n // 4 - b // 2, 0.5), (3 * n // 4 - b // 2, 0.001)):
            inb = ((cz[:, 0] > x0) & (cz[:, 0] < x0 + b) & (cz[:, 1] > n / 2 - b / 2)
                   & (cz[:, 1] < n / 2 + b / 2) & (cz[:, 2] > z1 - b) & (cz[:, 2] < z1))
            sig[inb] = s
    elif name == "C4":
        # 0.1 S/m plate, 2 cells thick, dipping 30 degrees along x under the air
        xc, zc = n / 2, z_if - max(2, n // 8)
        d = (cz[:, 2] - zc) * np.cos(np.pi / 6) - (cz[:, 0] - xc) * np.sin(np.pi / 6)
        inp = ((np.abs(d) < 1.0) & (np.abs(cz[:, 0] - xc) < n / 4)
               & (np.abs(cz[:, 1] - n / 2) < n / 4) & (cz[:, 2] < z_if))
        sig[inp] = 0.1
    elif name == "C5":
        z = cz[:, 2]
        sig = np.where(z > z_if - n / 6, 0.001, np.where(z > z_if - n / 2, 0.05, 0.01))
        rng = np.random.default_rng(3)
        for _ in range(3):
            c = rng.uniform(0.2, 0.8, 3) * np.array([n, n, z_if])
            s = rng.uniform(2, max(3, n / 8))
            inb = np.all(np.abs(cz - c) < s, axis=1) & (cz[:, 2] < z_if)
            sig[inb] = rng.uniform(0.1, 1.0)
    sig[air] = spec.sigma_air
    return np.log(sig)


def build_config(name: str, n: int | None = None, device: bool = False):
    """BASELINE config `name` (n overrides the mesh size); device=True builds
    the topology and K on the GPU (rba_box_generate)."""
    spec, meta = config_spec(name, n)
    m_true = config_true_model(name, spec)
    prob = build_box_problem(spec, m_true=m_true, device=device)
    return prob, meta
