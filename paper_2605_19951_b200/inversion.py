"""Drop-in for rbainv.inversion (/root/reference/pkg/src/rbainv/inversion.py).

The GN model update solves, matrix-free,

    | [ W_d J        ]        [ W_d (d(m) - d_obs)    ] |
    | [ sqrt(l) R    ] dm  +  [ sqrt(l) R (m - m_ref) ] |_2        (:1-13)

with LSQR.  ``lsqr_device`` restates SciPy's ``lsqr`` recurrences
(scipy/sparse/linalg/_isolve/lsqr.py:97, the routine ``_augmented_lsqr``
calls at :153) with every vector in HBM: J v / J^T w are the device
operators, R / R^T the device SpMV, and the vector updates and norms are the
deterministic K12 kernels; only the scalar recurrences run on the host.
The Armijo line search, cooling and bookkeeping (:179-307) are host control
flow, as in the reference.

Deviation (documented): the reference rebuilds the Jacobian operator after a
rejected line search without re-activating the cache and then raises
"cache has moved".  Here the operator constructor re-activates
the current model's factorisations, so the loop continues.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .forward import forward_device
from .problem import Model
from .regularization import RegOperator, build_reg, reg_value_grad
from .sensitivity import JacobianOperator
from .shifted import ShiftedFactorCache, PoleWorkerPool

__all__ = ["LsqrConfig", "InversionConfig", "IterationRecord", "InversionState",
           "LineSearchResult", "chi_squared", "default_lambda0", "gn_step", "line_search",
           "run_inversion", "lsqr_device"]


@dataclass(frozen=True)
class LsqrConfig:
    tol: float = 1e-3
    max_iters: int = 50


@dataclass(frozen=True)
class InversionConfig:
    lambda0: float | None = None
    chi2_target: float = 1.0
    max_gn: int = 30
    tol_outer: float = 1e-3
    lsqr: LsqrConfig = field(default_factory=LsqrConfig)
    c1: float = 1e-4
    eta_min: float = 2.0 ** -6
    lambda_min_factor: float = 2.0 ** -20
    quad_refine: bool = True
    workers: int = 1
    m0: np.ndarray | None = None


@dataclass
class IterationRecord:
    nu: int
    phi: float
    misfit: float
    reg_value: float
    chi2: float
    lam: float
    eta: float
    accepted: bool
    lsqr_iters: int
    lsqr_istop: int
    wall_ms: float
    factorizations: int
    solves: int
    phi_evals: int
    phi_before: float
    directional_slope: float

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k in self.__dataclass_fields__}


@dataclass
class InversionState:
    model: Model
    lam: float
    nu: int = 0
    phi: float = np.nan
    chi2: float = np.nan
    history: list = field(default_factory=list)
    diagnostic: str = ""
    counters: dict = field(default_factory=dict)


@dataclass
class LineSearchResult:
    eta: float
    accepted: bool
    phi: float
    n_evals: int


def chi_squared(data, d_pred: np.ndarray) -> float:
    if d_pred.size != data.size:
        raise ValueError("prediction length does not match data")
    r = data.weights * (d_pred - data.d_obs)
    return float(r @ r) / data.size


def default_lambda0(problem, data, reg: RegOperator, d_start: np.ndarray, model) -> float:
    misfit = float(np.sum((data.weights * (d_start - data.d_obs)) ** 2))
    pert = np.log(10.0) * np.sin(np.arange(model.cell_count, dtype=float))
    r_pert, _ = reg_value_grad(reg, Model(model.m_ref + pert, model.m_ref))
    return misfit / max(1.0, 2.0 * r_pert)


def _sym_ortho(a, b):
    """SciPy's stable Givens rotation (lsqr.py _sym_ortho)."""
    if b == 0:
        return np.sign(a), 0, abs(a)
    elif a == 0:
        return 0, np.sign(b), abs(b)
    elif abs(b) > abs(a):
        tau = a / b
        s = np.sign(b) / math.sqrt(1 + tau * tau)
        c = s * tau
        r = b / s
    else:
        tau = b / a
        c = np.sign(a) / math.sqrt(1 + tau * tau)
        s = c * tau
        r = a / c
    return c, s, r


class _AugmentedOp:
    """[W J ; sqrt(l) R] on device vectors (inversion.py:143-147)."""

    def __init__(self, opr: JacobianOperator, R_rows: int, W: torch.Tensor, sql: float):
        self.opr = opr
        self.eng = opr.engine
        self.n_data = W.numel()
        self.R_rows = R_rows
        self.W = W
        self.sql = sql
        self.shape = (self.n_data + R_rows, opr.shape[1])
        dev = W.device
        self._tmp_d = torch.empty(self.n_data, dtype=torch.float64, device=dev)

    def matvec(self, v, out):
        jv = self.opr.jvp_d(v)
        self.eng.mul(self.W, jv, out[:self.n_data])
        self.eng.reg_apply(v, out[self.n_data:], alpha=self.sql)
        return out

    def rmatvec(self, u, out):
        self.eng.mul(self.W, u[:self.n_data], self._tmp_d)
        jt = self.opr.vjp_d(self._tmp_d)
        out.copy_(jt)
        self.eng.reg_apply(u[self.n_data:], out, alpha=self.sql, transpose=True,
                           accumulate=True)
        return out


def lsqr_device(A: _AugmentedOp, b: torch.Tensor, atol: float, btol: float, iter_lim: int,
                conlim: float = 1e8):
    """SciPy lsqr (damp=0, x0=None), vectors on the device.  Returns (x, istop, itn)."""
    eng = A.eng
    m, n = A.shape
    dev = b.device
    eps = np.finfo(np.float64).eps
    itn, istop = 0, 0
    ctol = 1 / conlim if conlim > 0 else 0
    anorm = acond = ddnorm = res2 = xnorm = xxnorm = z = 0.0
    cs2, sn2 = -1.0, 0.0
    u = b.clone()
    bnorm = math.sqrt(eng.dot(u, u))
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    beta = bnorm
    v = torch.zeros(n, dtype=torch.float64, device=dev)
    tmp_m = torch.empty(m, dtype=torch.float64, device=dev)
    tmp_n = torch.empty(n, dtype=torch.float64, device=dev)
    alfa = 0.0
    if beta > 0:
        eng.axpby(1 / beta, u, 0.0, None, u)
        A.rmatvec(u, v)
        alfa = math.sqrt(eng.dot(v, v))
    if alfa > 0:
        eng.axpby(1 / alfa, v, 0.0, None, v)
    w = v.clone()
    rhobar, phibar = alfa, beta
    arnorm = alfa * beta
    if arnorm == 0:
        return x, istop, itn
    while itn < iter_lim:
        itn += 1
        A.matvec(v, tmp_m)
        eng.axpby(1.0, tmp_m, -alfa, u, u)
        beta = math.sqrt(eng.dot(u, u))
        if beta > 0:
            eng.axpby(1 / beta, u, 0.0, None, u)
            anorm = math.sqrt(anorm ** 2 + alfa ** 2 + beta ** 2)
            A.rmatvec(u, tmp_n)
            eng.axpby(1.0, tmp_n, -beta, v, v)
            alfa = math.sqrt(eng.dot(v, v))
            if alfa > 0:
                eng.axpby(1 / alfa, v, 0.0, None, v)
        rhobar1 = rhobar
        psi = 0.0
        cs, sn, rho = _sym_ortho(rhobar1, beta)
        theta = sn * alfa
        rhobar = -cs * alfa
        phi = cs * phibar
        phibar = sn * phibar
        tau = sn * phi
        t1 = phi / rho
        t2 = -theta / rho
        wn2 = eng.lsqr_xw(t1, t2, v, w, x)        # |w|^2 before update; x += t1 w; w = v + t2 w
        ddnorm = ddnorm + wn2 / (rho * rho)
        delta = sn2 * rho
        gambar = -cs2 * rho
        rhs = phi - delta * z
        zbar = rhs / gambar
        xnorm = math.sqrt(xxnorm + zbar ** 2)
        gamma = math.sqrt(gambar ** 2 + theta ** 2)
        cs2 = gambar / gamma
        sn2 = theta / gamma
        z = rhs / gamma
        xxnorm = xxnorm + z ** 2
        acond = anorm * math.sqrt(ddnorm)
        res1 = phibar ** 2
        res2 = res2 + psi ** 2
        rnorm = math.sqrt(res1 + res2)
        arnorm = alfa * abs(tau)
        test1 = rnorm / bnorm
        test2 = arnorm / (anorm * rnorm + eps)
        test3 = 1 / (acond + eps)
        t1 = test1 / (1 + anorm * xnorm / bnorm)
        rtol = btol + atol * anorm * xnorm / bnorm
        if itn >= iter_lim:
            istop = 7
        if 1 + test3 <= 1:
            istop = 6
        if 1 + test2 <= 1:
            istop = 5
        if 1 + t1 <= 1:
            istop = 4
        if test3 <= ctol:
            istop = 3
        if test2 <= atol:
            istop = 2
        if test1 <= rtol:
            istop = 1
        if istop != 0:
            break
    return x, istop, itn


def _device_reg(opr, reg: RegOperator):
    """Upload R (LSQR's square root) and L (reg_value_grad, the gradient term)
    once per (engine, regulariser)."""
    eng = getattr(opr, "engine", opr)
    if getattr(eng, "_reg_obj", None) is not reg:
        eng.set_reg(reg.R_factor)
        eng.set_reg_L(reg.L)
        eng._reg_obj = reg
    return eng.reg_rows


def reg_value_grad_device(eng, reg: RegOperator, r: torch.Tensor):
    """regularization.py:71-75 on the device for r = m - m_ref (device):
    returns (1/2 r^T L r, L r as a device tensor)."""
    _device_reg(eng, reg)
    Lr = torch.empty_like(r)
    eng.reg_L_apply(r, Lr)
    return 0.5 * eng.dot(r, Lr), Lr


def _augmented_lsqr(opr: JacobianOperator, reg: RegOperator, data, d_pred, model, lam: float,
                    lsqr_cfg: LsqrConfig):
    """inversion.py:133-155 on the device; returns (dm, itn, istop)."""
    x, itn, istop = _augmented_lsqr_d(opr, reg, data, d_pred, model, lam, lsqr_cfg)
    return x.cpu().numpy(), itn, istop


def _augmented_lsqr_d(opr: JacobianOperator, reg: RegOperator, data, d_pred, model, lam: float,
                      lsqr_cfg: LsqrConfig, W: torch.Tensor | None = None,
                      dobs: torch.Tensor | None = None, r: torch.Tensor | None = None):
    """Same, with dm left on the device (the GN driver's path)."""
    if not isinstance(opr, JacobianOperator):
        raise TypeError("the device LSQR needs the device JacobianOperator")
    eng = opr.engine
    dev = eng.device
    R_rows = _device_reg(opr, reg)
    if W is None:
        W = torch.as_tensor(np.asarray(data.weights, dtype=float), device=dev)
    sql = float(np.sqrt(lam))
    A = _AugmentedOp(opr, R_rows, W, sql)
    n_data = W.numel()
    b = torch.empty(n_data + R_rows, dtype=torch.float64, device=dev)
    dp = torch.as_tensor(np.asarray(d_pred, dtype=float) if not isinstance(d_pred, torch.Tensor)
                         else d_pred, device=dev, dtype=torch.float64)
    if dobs is None:
        dobs = torch.as_tensor(np.asarray(data.d_obs, dtype=float), device=dev)
    eng.axpby(1.0, dp, -1.0, dobs, b[:n_data])
    eng.mul(W, b[:n_data], b[:n_data], alpha=-1.0)
    if r is None:
        r = torch.as_tensor(np.asarray(model.m - model.m_ref, dtype=float), device=dev)
    eng.reg_apply(r, b[n_data:], alpha=-sql)
    x, istop, itn = lsqr_device(A, b, lsqr_cfg.tol, lsqr_cfg.tol, lsqr_cfg.max_iters)
    return x, int(itn), int(istop)


def gn_step(state: InversionState, problem, approx, reg: RegOperator, data,
            cache: ShiftedFactorCache, lsqr_cfg: LsqrConfig | None = None,
            pool: PoleWorkerPool | None = None, opr: JacobianOperator | None = None,
            d_pred: np.ndarray | None = None):
    """inversion.py:158-176: one linearised update; returns (dm, lsqr_iters)."""
    lsqr_cfg = lsqr_cfg or LsqrConfig()
    if opr is None:
        opr = JacobianOperator(problem, state.model, approx, cache, pool)
    if d_pred is None:
        d_pred = opr.engine.forward().cpu().numpy()
    dm, itn, istop = _augmented_lsqr(opr, reg, data, d_pred, state.model, state.lam, lsqr_cfg)
    state.counters["last_lsqr_istop"] = istop
    return dm, itn


def line_search(phi0: float, directional_slope: float, phi_evaluator, c1: float = 1e-4,
                eta_min: float = 2.0 ** -6, quad_refine: bool = True) -> LineSearchResult:
    """inversion.py:179-205 (identical control flow)."""
    eta = 1.0
    n_evals = 0
    quad_tried = False
    while eta >= eta_min:
        phi = phi_evaluator(eta)
        n_evals += 1
        if phi <= phi0 + c1 * eta * directional_slope:
            return LineSearchResult(eta, True, phi, n_evals)
        if quad_refine and not quad_tried:
            quad_tried = True
            denom = 2.0 * (phi - phi0 - directional_slope * eta)
            if denom > 0 and directional_slope < 0:
                eta_q = -directional_slope * eta * eta / denom
                eta_q = min(max(eta_q, eta_min), 0.9 * eta)
                if eta_q < eta:
                    phi_q = phi_evaluator(eta_q)
                    n_evals += 1
                    if phi_q <= phi0 + c1 * eta_q * directional_slope:
                        return LineSearchResult(eta_q, True, phi_q, n_evals)
        eta *= 0.5
    return LineSearchResult(eta_min, False, phi0, n_evals)


class GNDriver:
    """State of run_inversion (inversion.py:208-307) split so that one GN
    iteration can be timed on its own (bench.py)."""

    def __init__(self, problem, data, approx, cfg: InversionConfig | None = None,
                 cache: ShiftedFactorCache | None = None, reg: RegOperator | None = None):
        self.cfg = cfg or InversionConfig()
        self.cache = cache or ShiftedFactorCache()
        self.pool = PoleWorkerPool(self.cfg.workers)
        self.problem, self.data, self.approx = problem, data, approx
        self.reg = reg or build_reg(problem.grid)
        ref = problem.reference_model()
        m_start = self.cfg.m0 if self.cfg.m0 is not None else ref.m
        self.model = Model(np.asarray(m_start, dtype=float), ref.m_ref)
        self.W = data.weights
        self.n_data = data.size
        self._dv_key = None
        self.g_tag, self.d_pred, self.misfit, self.reg_val = self.forward_at(self.model)
        cfg = self.cfg
        self.lam = cfg.lambda0 if cfg.lambda0 is not None else default_lambda0(
            problem, data, self.reg, self.d_pred.cpu().numpy(), self.model)
        self.lam_min = self.lam * cfg.lambda_min_factor
        self.phi = self.misfit + self.lam * self.reg_val
        self.chi2 = 2.0 * self.misfit / self.n_data
        self.state = InversionState(model=self.model, lam=self.lam, phi=self.phi, chi2=self.chi2)
        self.increase_streak = 0

    def _vectors(self, eng):
        """W, W*W and d_obs resident on the device (refreshed when the caller
        hands in new data arrays)."""
        key = (id(eng), id(self.W), id(self.data.d_obs))
        if self._dv_key != key:
            dev = eng.device
            self._W_d = torch.as_tensor(np.asarray(self.W, dtype=float), device=dev)
            self._W2_d = torch.empty_like(self._W_d)
            eng.mul(self._W_d, self._W_d, self._W2_d)
            self._dobs_d = torch.as_tensor(np.asarray(self.data.d_obs, dtype=float), device=dev)
            self._tmp_d = torch.empty_like(self._W_d)
            self._dv_key = key
        return self._W_d, self._W2_d, self._dobs_d

    def forward_at(self, mdl: Model):
        """inversion.py:223-228 with every vector operation on the device:
        d (kept in HBM), misfit 1/2|W(d - d_obs)|^2 and reg_value_grad
        (1/2 r^T L r, device SpMV)."""
        d = forward_device(self.problem, mdl, self.approx, self.cache)
        eng = self.cache.engine
        W, _, dobs = self._vectors(eng)
        t = self._tmp_d
        eng.axpby(1.0, d, -1.0, dobs, t)
        eng.mul(W, t, t)
        mis = 0.5 * eng.dot(t, t)
        r = torch.as_tensor(np.asarray(mdl.m - mdl.m_ref, dtype=float), device=eng.device)
        rv, _ = reg_value_grad_device(eng, self.reg, r)
        return mdl.version_tag(), d, mis, rv

    def iterate(self, nu: int) -> bool:
        """One GN iteration; returns False when the loop must stop."""
        cfg, state, cache = self.cfg, self.state, self.cache
        model = self.model
        t0 = time.perf_counter()
        counters0 = cache.counters.snapshot()
        opr = JacobianOperator(self.problem, model, self.approx, cache, self.pool)
        eng = opr.engine
        dev = eng.device
        W, W2, dobs = self._vectors(eng)
        # gradient (inversion.py:250): J^T (W*W*(d - d_obs)) + lambda L (m - m_ref)
        residual = torch.empty_like(W)
        eng.axpby(1.0, self.d_pred, -1.0, dobs, residual)
        eng.mul(W2, residual, residual)
        r = torch.as_tensor(np.asarray(model.m - model.m_ref, dtype=float), device=dev)
        _, Lr = reg_value_grad_device(eng, self.reg, r)
        grad = opr.vjp_d(residual)
        eng.axpby(1.0, grad, self.lam, Lr, grad)
        dm_d, lsqr_iters, istop = _augmented_lsqr_d(opr, self.reg, self.data, self.d_pred, model,
                                                    self.lam, cfg.lsqr, W=W, dobs=dobs, r=r)
        slope = eng.dot(grad, dm_d)
        dm = dm_d.cpu().numpy()
        evals: dict[float, tuple] = {}

        def phi_eval(eta: float) -> float:
            trial = Model(model.m + eta * dm, model.m_ref)
            out = self.forward_at(trial)
            evals[eta] = (trial, out)
            return out[2] + self.lam * out[3]

        ls = line_search(self.phi, slope, phi_eval, c1=cfg.c1, eta_min=cfg.eta_min,
                         quad_refine=cfg.quad_refine)
        wall_ms = (time.perf_counter() - t0) * 1e3
        counters1 = cache.counters.snapshot()
        phi_before = self.phi
        if ls.accepted:
            self.model, (self.g_tag, self.d_pred, self.misfit, self.reg_val) = evals[ls.eta]
            state.model = self.model
            new_phi = self.misfit + self.lam * self.reg_val
            self.chi2 = 2.0 * self.misfit / self.n_data
            self.increase_streak = self.increase_streak + 1 if new_phi > self.phi else 0
            rel_decrease = (self.phi - new_phi) / max(abs(self.phi), 1e-300)
            self.phi = new_phi
        else:
            rel_decrease = 0.0
        state.history.append(IterationRecord(
            nu=nu, phi=self.phi, misfit=self.misfit, reg_value=self.reg_val, chi2=self.chi2,
            lam=self.lam, eta=ls.eta if ls.accepted else 0.0, accepted=ls.accepted,
            lsqr_iters=lsqr_iters, lsqr_istop=istop, wall_ms=wall_ms,
            factorizations=counters1["factorizations"] - counters0["factorizations"],
            solves=counters1["solves"] - counters0["solves"],
            phi_evals=ls.n_evals, phi_before=phi_before, directional_slope=slope))
        state.phi, state.chi2, state.lam = self.phi, self.chi2, self.lam
        if self.increase_streak >= 3:
            state.diagnostic = "divergence guard: objective rose on 3 consecutive accepted steps"
            return False
        if not ls.accepted or rel_decrease < cfg.tol_outer:
            self.lam *= 0.5
            if self.lam < self.lam_min:
                state.diagnostic = "lambda floor reached"
                state.lam = self.lam
                return False
            self.phi = self.misfit + self.lam * self.reg_val
            state.lam = self.lam
            state.phi = self.phi
        return True


def run_inversion(problem, data, approx, cfg: InversionConfig | None = None,
                  cache: ShiftedFactorCache | None = None, reg: RegOperator | None = None
                  ) -> InversionState:
    """inversion.py:208-307"""
    drv = GNDriver(problem, data, approx, cfg, cache, reg)
    state = drv.state
    for nu in range(1, drv.cfg.max_gn + 1):
        state.nu = nu
        if drv.chi2 <= drv.cfg.chi2_target:
            state.diagnostic = "chi2 target reached"
            break
        if not drv.iterate(nu):
            break
    else:
        state.diagnostic = state.diagnostic or "max Gauss-Newton iterations"
    if drv.chi2 <= drv.cfg.chi2_target:
        state.diagnostic = "chi2 target reached"
    state.counters.update(drv.cache.counters.snapshot())
    return state
