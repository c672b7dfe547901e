"""CPU ORACLE -- test infrastructure only, never the product path.

A plain NumPy/SciPy restatement of the reference's shifted-solve
Gauss-Newton path (arXiv 2605.19951 analog, /root/reference/pkg/src/rbainv).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module, and only as the checker / the timed CPU
reference.  The product (paper_2605_19951_b200) never imports it.

Pinning: every function below is checked against golden vectors produced by
the unmodified reference itself (``tests/golden/make_golden.py`` imports
/root/reference in the build container; outputs committed as .npz) -- see
tests/test_oracle_golden.py.

Each function cites the reference file:line it restates.  Multi-source
problems (S transmitter loops; the reference has a single ``f``) are
composed exactly as SURVEY.md §7 prescribes: stacked data
[source][channel][receiver], jvp stacked per source, vjp summed over sources
in ascending order.
"""

from __future__ import annotations

import hashlib
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.linalg as la
import scipy.sparse as sp
import scipy.sparse.linalg as spla

__all__ = [
    "assemble_M", "dM_contract", "PoleFactors", "factorize_all_poles",
    "solve_all_poles", "response_from_pole_solutions", "forward_response",
    "Jacobian", "adjoint_test", "build_reg", "face_root", "augmented_lsqr",
    "gn_step", "line_search", "make_dataset", "chi_squared", "version_tag",
]


def version_tag(m: np.ndarray) -> str:
    """mesh.py:84-85"""
    return hashlib.sha1(np.asarray(m, dtype=float).tobytes()).hexdigest()[:16]


def _scatter(problem):
    """mesh.py:319-323, 342-343 (cached COO pattern)."""
    if getattr(problem, "_scatter", None) is not None:
        return problem._scatter
    k = problem.cell_dofs.shape[1]
    rows = np.repeat(problem.cell_dofs, k, axis=1).ravel()
    cols = np.tile(problem.cell_dofs, (1, k)).ravel()
    keep = (rows >= 0) & (cols >= 0)
    cell_of = np.repeat(np.arange(problem.cell_dofs.shape[0]), k * k)[keep]
    problem._scatter = (rows[keep], cols[keep], keep, cell_of)
    return problem._scatter


def assemble_M(problem, m: np.ndarray) -> sp.csr_matrix:
    """mesh.py:348-355: M = sum_c e^{m_c} M_c via COO -> CSR."""
    rows, cols, keep, cell_of = _scatter(problem)
    vals = problem.mass_local.ravel()[keep] * np.exp(m)[cell_of]
    N = problem.K.shape[0]
    return sp.coo_matrix((vals, (rows, cols)), shape=(N, N)).tocsr()


def dM_contract(problem, m: np.ndarray, g: np.ndarray) -> sp.csc_matrix:
    """mesh.py:358-370: column c = e^{m_c} (M_c g|_c) on the cell dofs."""
    dofs = problem.cell_dofs
    gl = np.where(dofs >= 0, g[np.maximum(dofs, 0)], 0.0)
    local = np.einsum("pij,pj->pi", problem.mass_local, gl) * np.exp(m)[:, None]
    P, k = dofs.shape
    cols = np.repeat(np.arange(P), k)
    rows = dofs.ravel()
    keep = rows >= 0
    return sp.coo_matrix((local.ravel()[keep], (rows[keep], cols.ravel()[keep])),
                         shape=(problem.K.shape[0], P)).tocsc()


class PoleFactors:
    """shifted.py:44-122: SuperLU factor per pole of A_i = K - xi_i M(m),
    keyed by the model tag; counters as CacheCounters (shifted.py:64-70)."""

    def __init__(self, permc_spec: str = "COLAMD", workers: int = 1):
        self.permc_spec = permc_spec     # SuperLU ordering (reference default: COLAMD)
        # PoleWorkerPool (shifted.py:129-155): worker p owns poles i mod W;
        # SuperLU releases the GIL, so threads factorise/solve poles in parallel
        self.workers = max(1, int(workers))
        self._pool = ThreadPoolExecutor(self.workers) if self.workers > 1 else None
        self.tag = None
        self.lu = {}
        self.A = {}
        self.factorizations = 0
        self.solves = 0

    def activate(self, tag):
        if tag != self.tag:
            self.lu = {}
            self.A = {}
            self.tag = tag

    def solve(self, i, rhs, trans="N"):
        self.solves += 1
        return self.lu[i].solve(np.asarray(rhs, dtype=complex), trans=trans)

    def map_poles(self, fn, count):
        """shifted.py:140-155: pole-indexed results, worker p runs i = p, p+W, ..."""
        if self._pool is None:
            return [fn(i) for i in range(count)]
        W = self.workers

        def run(p):
            return [(i, fn(i)) for i in range(p, count, W)]
        out = [None] * count
        for chunk in self._pool.map(run, range(W)):
            for i, r in chunk:
                out[i] = r
        return out


def factorize_all_poles(problem, m, poles, fac: PoleFactors):
    """shifted.py:158-173"""
    fac.activate(version_tag(m))
    missing = [i for i in range(len(poles)) if i not in fac.lu]
    if not missing:
        return
    M = assemble_M(problem, m).astype(complex).tocsc()
    K = problem.K.astype(complex).tocsc()

    def one(k):
        i = missing[k]
        A = K - poles[i] * M
        try:
            lu = spla.splu(A.tocsc(), permc_spec=fac.permc_spec)
        except Exception as exc:  # shifted.py:55-56
            raise RuntimeError(f"factorization of shifted matrix failed: {exc}") from exc
        return i, lu, A.tocsr()
    for i, lu, A in fac.map_poles(one, len(missing)):
        fac.lu[i] = lu
        fac.A[i] = A
        fac.factorizations += 1


def solve_all_poles(problem, m, poles, rhs, fac: PoleFactors, check_residuals=False):
    """shifted.py:176-199: (m, N) complex; rhs may be (N,) or (N, S)."""
    factorize_all_poles(problem, m, poles, fac)
    rhs = np.asarray(rhs)
    out = []
    nrm = np.linalg.norm(rhs)
    gs = fac.map_poles(lambda i: fac.solve(i, rhs), len(poles))
    for i in range(len(poles)):
        g = gs[i]
        if check_residuals and nrm > 0:
            res = np.linalg.norm(fac.A[i] @ g - rhs) / nrm
            if res > 1e-8:
                raise RuntimeError(f"pole {i}: relative residual {res:.3e} exceeds 1e-8")
        out.append(g)
    return np.array(out)


def response_from_pole_solutions(Q, residues, g):
    """forward.py:46-64 (data path): D[j, r] = sum_i 2 Re(alpha_ij (Q g_i)_r),
    ascending pole order, flattened channel-major.  g is (m, N)."""
    m, K_t = residues.shape
    D = np.zeros((K_t, Q.shape[0]))
    for i in range(m):
        D += 2.0 * np.real(np.outer(residues[i], Q @ g[i]))
    return D.ravel()


def _sources(problem):
    src = getattr(problem, "sources", None)
    if src is None:
        return np.asarray(problem.f, dtype=float)[None, :]
    return np.asarray(src, dtype=float)


def forward_response(problem, m, poles, residues, fac: PoleFactors):
    """forward.py:67-75, stacked over sources: returns (data, g) with
    g of shape (m, N, S)."""
    F = _sources(problem)
    g = solve_all_poles(problem, m, poles, F.T, fac)          # (m, N, S)
    data = np.concatenate([response_from_pole_solutions(problem.Q, residues, g[:, :, s])
                           for s in range(F.shape[0])])
    return data, g


class Jacobian:
    """sensitivity.py:35-116 (JacobianOperator), source-stacked."""

    def __init__(self, problem, m, poles, residues, fac: PoleFactors, g=None):
        self.problem, self.m = problem, np.asarray(m, dtype=float)
        self.poles, self.residues, self.fac = poles, residues, fac
        if g is None:
            _, g = forward_response(problem, m, poles, residues, fac)
        self.g = g
        self.S = g.shape[2]
        self.dM = [[dM_contract(problem, self.m, g[i, :, s]) for i in range(len(poles))]
                   for s in range(self.S)]
        self.n_chan = residues.shape[1]
        self.n_recv = problem.Q.shape[0]
        self.shape = (self.S * self.n_chan * self.n_recv, problem.cell_dofs.shape[0])

    def jvp(self, v):
        """sensitivity.py:65-79"""
        v = np.asarray(v, dtype=float)
        out = []
        for s in range(self.S):
            D = np.zeros((self.n_chan, self.n_recv))
            qs = self.fac.map_poles(
                lambda i: self.problem.Q @ self.fac.solve(i, self.dM[s][i] @ v), len(self.poles))
            for i in range(len(self.poles)):
                D += 2.0 * np.real(self.poles[i] * np.outer(self.residues[i], qs[i]))
            out.append(D.ravel())
        return np.concatenate(out)

    def vjp(self, w):
        """sensitivity.py:81-97; sources summed in ascending order."""
        w = np.asarray(w, dtype=float).reshape(self.S, self.n_chan, self.n_recv)
        total = np.zeros(self.shape[1])
        for s in range(self.S):
            Qt_w = self.problem.Q.T @ w[s].T
            out = np.zeros(self.shape[1])
            ts = self.fac.map_poles(
                lambda i: self.dM[s][i].T @ self.fac.solve(i, Qt_w @ self.residues[i], trans="T"),
                len(self.poles))
            for i in range(len(self.poles)):
                out += 2.0 * np.real(self.poles[i] * ts[i])
            total = total + out if s else out
        return total


def adjoint_test(opr, trials=20, seed=0):
    """sensitivity.py:175-188"""
    rng = np.random.default_rng(seed)
    worst = 0.0
    for _ in range(trials):
        v = rng.standard_normal(opr.shape[1])
        w = rng.standard_normal(opr.shape[0])
        lhs = float(opr.jvp(v) @ w)
        rhs = float(v @ opr.vjp(w))
        worst = max(worst, abs(lhs - rhs) / max(abs(lhs), abs(rhs)))
    return worst


def build_reg(grid, dense_chol=True):
    """regularization.py:40-68: D, lumped face mass, L = D Mdiv^-1 D^T +
    eps diag(meas), and R with R^T R = L (dense Cholesky, as the reference)."""
    P = grid.cell_measure.size
    F = grid.face_cells.shape[0]
    rows = grid.face_cells.ravel()
    cols = np.repeat(np.arange(F), 2)
    vals = np.tile([1.0, -1.0], F) * np.repeat(grid.face_measure, 2)
    D = sp.coo_matrix((vals, (rows, cols)), shape=(P, F)).tocsr()
    mdiv = grid.cell_measure[grid.face_cells].mean(axis=1)
    L_div = (D @ sp.diags(1.0 / mdiv) @ D.T).tocsr()
    eps = 1e-8 * (L_div.diagonal().sum() / P if F else 1.0)
    L = (L_div + eps * sp.diags(grid.cell_measure)).tocsr()
    R = sp.csr_matrix(la.cholesky(L.toarray(), lower=False)) if dense_chol else None
    return dict(D=D, mdiv=mdiv, L=L, L_div=L_div, R=R, eps=eps)


def face_root(reg, grid):
    """R~ = [diag(mdiv)^-1/2 D^T ; sqrt(eps) diag(sqrt(meas))],
    R~^T R~ = L exactly in exact arithmetic."""
    top = sp.diags(1.0 / np.sqrt(reg["mdiv"])) @ reg["D"].T
    bot = sp.diags(np.sqrt(reg["eps"] * grid.cell_measure))
    return sp.vstack([top, bot]).tocsr()


def chi_squared(weights, d_obs, d_pred):
    """inversion.py:109-114"""
    r = weights * (d_pred - d_obs)
    return float(r @ r) / d_obs.size


def augmented_lsqr(opr, R, weights, d_obs, d_pred, m, m_ref, lam, tol, max_iters):
    """inversion.py:133-155 (SciPy lsqr with atol=btol=tol, iter_lim=max_iters)."""
    n_data = d_obs.size
    P = m.size
    W = weights
    sql = np.sqrt(lam)

    def matvec(v):
        return np.concatenate([W * opr.jvp(v), sql * (R @ v)])

    def rmatvec(u):
        return opr.vjp(W * u[:n_data]) + sql * (R.T @ u[n_data:])

    op = spla.LinearOperator((n_data + R.shape[0], P), matvec=matvec, rmatvec=rmatvec,
                             dtype=float)
    b = -np.concatenate([W * (d_pred - d_obs), sql * (R @ (m - m_ref))])
    x, istop, itn, *_ = spla.lsqr(op, b, atol=tol, btol=tol, iter_lim=max_iters)
    return x, int(itn), int(istop)


def line_search(phi0, slope, phi_evaluator, c1=1e-4, eta_min=2.0 ** -6, quad_refine=True):
    """inversion.py:179-205 (Armijo halving + one quadratic candidate)."""
    eta, n_evals, quad_tried = 1.0, 0, False
    while eta >= eta_min:
        phi = phi_evaluator(eta)
        n_evals += 1
        if phi <= phi0 + c1 * eta * slope:
            return eta, True, phi, n_evals
        if quad_refine and not quad_tried:
            quad_tried = True
            denom = 2.0 * (phi - phi0 - slope * eta)
            if denom > 0 and slope < 0:
                eta_q = -slope * eta * eta / denom
                eta_q = min(max(eta_q, eta_min), 0.9 * eta)
                if eta_q < eta:
                    phi_q = phi_evaluator(eta_q)
                    n_evals += 1
                    if phi_q <= phi0 + c1 * eta_q * slope:
                        return eta_q, True, phi_q, n_evals
        eta *= 0.5
    return eta_min, False, phi0, n_evals


def gn_step(problem, m, m_ref, poles, residues, R, weights, d_obs, lam, tol, max_iters,
            fac: PoleFactors):
    """inversion.py:158-176: one linearised update (dm, itn, istop, d_pred)."""
    d_pred, g = forward_response(problem, m, poles, residues, fac)
    opr = Jacobian(problem, m, poles, residues, fac, g=g)
    dm, itn, istop = augmented_lsqr(opr, R, weights, d_obs, d_pred, m, m_ref, lam,
                                    tol, max_iters)
    return dm, itn, istop, d_pred


def gn_iteration(problem, m, m_ref, poles, residues, R, L, weights, d_obs, lam, iters,
                 fac: PoleFactors, d_pred=None, g=None, c1=1e-4, eta_min=2.0 ** -6):
    """One Gauss-Newton iteration of run_inversion (inversion.py:240-300):
    operator from the current g, gradient J^T(W^2 (d - d_obs)) + lam L (m - m_ref),
    LSQR (tol 0, `iters` iterations), Armijo line search whose every trial
    refactorises all poles (forward_at, inversion.py:223-228).  Returns
    (m_new, accepted, eta, n_evals, d_new, g_new)."""
    W = weights
    if d_pred is None or g is None:
        d_pred, g = forward_response(problem, m, poles, residues, fac)
    J = Jacobian(problem, m, poles, residues, fac, g=g)
    grad = J.vjp(W * W * (d_pred - d_obs)) + lam * (L @ (m - m_ref))
    dm, _, _ = augmented_lsqr(J, R, W, d_obs, d_pred, m, m_ref, lam, 0.0, iters)
    slope = float(grad @ dm)

    def phi_of(mm, d):
        r = mm - m_ref
        return 0.5 * float(np.sum((W * (d - d_obs)) ** 2)) + lam * 0.5 * float(r @ (L @ r))
    phi0 = phi_of(m, d_pred)
    evals = {}

    def ev(eta):
        mm = m + eta * dm
        d, gg = forward_response(problem, mm, poles, residues, fac)
        evals[eta] = (mm, d, gg)
        return phi_of(mm, d)
    eta, ok, _, n = line_search(phi0, slope, ev, c1=c1, eta_min=eta_min)
    if ok:
        mm, d, gg = evals[eta]
        return mm, True, eta, n, d, gg
    return m, False, eta, n, d_pred, g


def lsqr_floor(problem, m, poles, residues, R, weights, d_obs, lam, iters, orderings=(
        "COLAMD", "MMD_AT_PLUS_A"), m_ref=None, return_all=False):
    """The reference's own solver-to-solver floor on the GN update:
    relative difference of dm computed with two SuperLU orderings."""
    out = []
    for spec in orderings:
        fac = PoleFactors(spec)
        d, g = forward_response(problem, m, poles, residues, fac)
        J = Jacobian(problem, m, poles, residues, fac, g=g)
        dm, _, _ = augmented_lsqr(J, R, weights, d_obs, d, m, m if m_ref is None else m_ref,
                                  lam, 0.0, iters)
        out.append(dm)
    if return_all:
        return float(np.linalg.norm(out[0] - out[1]) / np.linalg.norm(out[0])), out
    return float(np.linalg.norm(out[0] - out[1]) / np.linalg.norm(out[0])), out[0]


def make_dataset(d_clean, eps_r, eps_a=None, seed=0):
    """synthetic.py:63-82 (noise model and seeded RNG)."""
    eps_a = eps_a if eps_a is not None else 1e-6 * np.max(np.abs(d_clean))
    sigma = np.abs(d_clean) * eps_r + eps_a
    rng = np.random.default_rng(seed)
    d_obs = d_clean + sigma * rng.standard_normal(d_clean.size)
    return d_obs, sigma
