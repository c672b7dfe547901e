"""Device engine: one `rba_ctx` (C ABI) bound to a problem and an approximant.

Owns the device-resident state of the shifted-solve path -- mesh operators,
the symbolic structure, the per-pole factorisations, pole solutions g_i and
work vectors -- and exposes the operations the reference's modules call:

* ``set_model``  -> M(m) assembly on the device (mesh.py:348-355)
* ``factor``     -> factorize_all_poles (shifted.py:158-173)
* ``forward``    -> solve_all_poles + response_from_pole_solutions
                    (shifted.py:176-199, forward.py:46-75)
* ``jvp``/``vjp``-> JacobianOperator actions (sensitivity.py:65-97)
* ``solve``      -> cache.solve (shifted.py:107-116)

Poles are sharded i -> rank (i mod G) like PoleWorkerPool (shifted.py:147-149);
per-pole partials are exchanged with ``parallel.gather_partials`` and summed
on every rank in ascending pole order, so results are bitwise identical for
any GPU count.  PyTorch is used only for device allocation, streams and the
collectives; every arithmetic step runs in libdrba.so kernels.
"""

from __future__ import annotations

import os

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from ._lib import check, ptr
from . import parallel

__all__ = ["Engine", "pattern_coords"]


def pattern_coords(problem):
    c = getattr(problem, "dof_coords", None)
    if c is None:
        return None
    return np.ascontiguousarray(c, dtype=np.float64)


class Engine:
    """Device state for one (problem, approximant) pair."""

    def __init__(self, problem, approx=None, device: int | None = None, leaf: int = 64,
                 comm: parallel.PoleComm | None = None, n_slots: int | None = None,
                 lazy_factors: bool = False):
        self.lib = _lib.load()
        if not torch.cuda.is_available():
            raise RuntimeError("the B200 shifted-solve path needs a CUDA device "
                               "(no CPU fallback)")
        self.comm = comm or parallel.PoleComm.current()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else device)
        self.stream = torch.cuda.current_stream(self.device)
        h = _lib.vp()
        # run on torch's current stream so torch ops (H2D copies, allocations,
        # collectives) and the library's kernels are ordered.  torch's default
        # stream is the legacy NULL stream, which must be passed as
        # cudaStreamLegacy (0x1): a NULL handle would make the library create
        # its own non-blocking stream.
        handle = self.stream.cuda_stream or 0x1
        check(self.lib.rba_ctx_create(self.device.index, _lib.vp(handle), _lib.C.byref(h)))
        self.ctx = h
        self.problem = problem
        self.N = int(problem.K.shape[0])
        self.P = int(problem.cell_dofs.shape[0]) if problem.cell_dofs is not None else 0
        K = sp.csr_matrix(problem.K)
        K.sort_indices()
        k = int(problem.cell_dofs.shape[1]) if self.P else 1
        cd = np.ascontiguousarray(problem.cell_dofs, dtype=np.int32) if self.P \
            else np.zeros((0, 1), np.int32)
        ml = np.ascontiguousarray(problem.mass_local, dtype=np.float64) if self.P \
            else np.zeros((0, 1, 1))
        coords = pattern_coords(problem)
        # keep every converted array referenced until the call returns
        kp = np.ascontiguousarray(K.indptr, dtype=np.int64)
        ki = np.ascontiguousarray(K.indices, dtype=np.int32)
        kx = np.ascontiguousarray(K.data, dtype=np.float64)
        check(self.lib.rba_set_mesh(self.ctx, self.N, self.P, k, ptr(cd), ptr(ml), ptr(kp),
                                    ptr(ki), ptr(kx), ptr(coords), int(os.environ.get("RBA_LEAF", leaf))))
        Q = sp.csr_matrix(problem.Q)
        self.Mr = int(Q.shape[0])
        qp = np.ascontiguousarray(Q.indptr, dtype=np.int64)
        qi = np.ascontiguousarray(Q.indices, dtype=np.int32)
        qx = np.ascontiguousarray(Q.data, dtype=np.float64)
        check(self.lib.rba_set_observation(self.ctx, self.Mr, ptr(qp), ptr(qi), ptr(qx)))
        F = problem.source_matrix() if hasattr(problem, "source_matrix") else \
            np.asarray(problem.f, dtype=float)[None, :]
        self.set_sources(F)
        self.approx = None
        self.model_tag = None
        self.factored = False
        self.g_valid = False
        self.reg_rows = 0
        if lazy_factors:
            self.set_option("lazy_factors", 1)
        if approx is not None:
            self.set_poles(approx)
        elif n_slots:
            self._set_dummy_poles(n_slots)

    # ------------------------------------------------------------------ setup
    def set_sources(self, F):
        F = np.atleast_2d(F)
        if F.shape[1] != self.N:
            raise ValueError("source vectors must have length N")
        self.S = F.shape[0]
        if np.iscomplexobj(F):
            Fc = np.ascontiguousarray(F, dtype=np.complex128)
            check(self.lib.rba_set_sources_complex(self.ctx, self.S, ptr(Fc.view(np.float64))))
        else:
            Fr = np.ascontiguousarray(F, dtype=np.float64)
            check(self.lib.rba_set_sources(self.ctx, self.S, ptr(Fr)))
        self.factored = False

    def set_poles(self, approx):
        poles = np.ascontiguousarray(approx.poles, dtype=np.complex128)
        res = np.ascontiguousarray(approx.residues, dtype=np.complex128)
        self.m = poles.size
        self.Kt = res.shape[1]
        self.local = self.comm.local_poles(self.m)
        loc = np.ascontiguousarray(self.local, dtype=np.int32)
        check(self.lib.rba_set_poles(self.ctx, self.m, ptr(poles.view(np.float64)), self.Kt,
                                     ptr(res.view(np.float64)), loc.size, ptr(loc)))
        self.approx = approx
        self.poles = poles
        self.residues = res
        self.factored = False
        self.g_valid = False
        nl = max(1, self.comm.n_max(self.m))
        dev = self.device
        self.qpart = torch.zeros((nl, self.S, max(self.Mr, 1)), dtype=torch.complex128, device=dev)
        self.tpart = torch.zeros((nl, self.P), dtype=torch.float64, device=dev)
        self.slot_of_pole = self.comm.slot_of_pole(self.m)
        if self.comm.world > 1:
            # every rank must round J v / J^T w the same way: receiver-Green
            # mode only if it fits on every rank (it depends on free memory)
            on = bool(self.info()["green"])
            if self.comm.agree_min(int(on)) == 0 and on:
                self.set_option("green", 0)

    def set_option(self, name: str, value: int):
        check(self.lib.rba_set_option(self.ctx, name.encode(), int(value)))

    def _set_dummy_poles(self, n):
        class _A:
            pass
        a = _A()
        a.poles = 1j * (np.arange(n) + 1.0)
        a.residues = np.zeros((n, 1), complex)
        self.set_poles(a)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.rba_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ model/factor
    def set_model(self, m, tag: str | None = None):
        if isinstance(m, torch.Tensor):
            mt = m.to(self.device, torch.float64).contiguous()
            check(self.lib.rba_set_model_d(self.ctx, ptr(mt)))
        else:
            mh = np.ascontiguousarray(m, dtype=np.float64)
            if mh.size != self.P:
                raise ValueError("model size does not match grid")
            check(self.lib.rba_set_model(self.ctx, ptr(mh)))
        self.model_tag = tag
        self.last_m = m                 # the model the current factors belong to
        self.factored = False
        self.g_valid = False

    def factor(self):
        check(self.lib.rba_factor(self.ctx))
        self.factored = True

    def factor_values(self, slot: int, values: np.ndarray):
        v = np.ascontiguousarray(values, dtype=np.complex128)
        check(self.lib.rba_factor_values(self.ctx, int(slot), ptr(v.view(np.float64))))

    def pattern(self, with_M: bool = False):
        n = _lib.i64()
        check(self.lib.rba_pattern(self.ctx, _lib.C.byref(n), None, None, None, None))
        nnz = n.value
        rows = np.empty(nnz, np.int32)
        cols = np.empty(nnz, np.int32)
        Kv = np.empty(nnz)
        Mv = np.empty(nnz) if with_M else None
        check(self.lib.rba_pattern(self.ctx, _lib.C.byref(n), ptr(rows), ptr(cols), ptr(Kv),
                                   ptr(Mv)))
        return rows, cols, Kv, Mv

    # ------------------------------------------------------------- operators
    TRANS = {"N": 0, "T": 1, "H": 2}

    @classmethod
    def _trans(cls, trans: str) -> int:
        """_Factor.solve's trans (shifted.py:58-61): 'N', 'T' (= 'N', A complex
        symmetric) or 'H' (conjugate transpose); anything else is an error."""
        try:
            return cls.TRANS[trans]
        except (KeyError, TypeError):
            raise ValueError(f"trans must be 'N', 'T' or 'H', got {trans!r}") from None

    def solve(self, slot: int, rhs: np.ndarray, trans: str = "N") -> np.ndarray:
        t = self._trans(trans)
        rhs = np.asarray(rhs, dtype=np.complex128)
        one = rhs.ndim == 1
        B = np.ascontiguousarray(rhs.reshape(self.N, -1).T)       # (nrhs, N) = col-major N x nrhs
        out = np.empty_like(B)
        check(self.lib.rba_solve(self.ctx, int(slot), ptr(B.view(np.float64)),
                                 ptr(out.view(np.float64)), B.shape[0], t))
        return out[0] if one else out.T.copy()

    def solve_d(self, slot: int, rhs: torch.Tensor, trans: str = "N") -> torch.Tensor:
        t = self._trans(trans)
        rhs = rhs.to(self.device, torch.complex128).contiguous()
        out = torch.empty_like(rhs)
        nrhs = 1 if rhs.dim() == 1 else rhs.shape[0]
        check(self.lib.rba_solve_d(self.ctx, int(slot), ptr(rhs), ptr(out), nrhs, t))
        return out

    def download_g(self, slot: int) -> np.ndarray:
        """g of a local slot as (N, S) complex in the original dof order."""
        out = np.empty((self.S, self.N), dtype=np.complex128)
        check(self.lib.rba_get_g(self.ctx, int(slot), ptr(out.view(np.float64))))
        return out.T.copy()

    def g_device(self, slot: int) -> torch.Tensor:
        """g of a local slot as a (S, N) complex device tensor, original order."""
        out = torch.empty((self.S, self.N), dtype=torch.complex128, device=self.device)
        check(self.lib.rba_get_g_d(self.ctx, int(slot), ptr(out)))
        return out

    def upload_g(self, slot: int, g: np.ndarray):
        """Replace g of a local slot by given pole solutions, (N,) or (N, S)."""
        g = np.asarray(g, dtype=np.complex128).reshape(self.N, -1)
        if g.shape[1] != self.S:
            raise ValueError(f"pole solutions need {self.S} source column(s)")
        h = np.ascontiguousarray(g.T)
        check(self.lib.rba_set_g(self.ctx, int(slot), ptr(h.view(np.float64))))

    def gather_fields(self) -> torch.Tensor:
        """g_i of ALL poles (m, S, N) on every rank: per-rank local fields,
        all-gathered (rank-major) and put in global pole order."""
        nmax = self.comm.n_max(self.m)
        loc = torch.zeros((nmax, self.S, self.N), dtype=torch.complex128, device=self.device)
        for slot in range(len(self.local)):
            loc[slot] = self.g_device(slot)
        allg = self._gather(loc)
        idx = torch.as_tensor(self.slot_of_pole.astype(np.int64), device=self.device)
        return allg.index_select(0, idx)

    def factor_stats(self, slot: int) -> dict:
        """Pivot-free LDL^T stability report of a local slot (rba_factor_stats)."""
        out = np.zeros(4)
        check(self.lib.rba_factor_stats(self.ctx, int(slot), ptr(out)))
        return {"max_abs_Lp": float(out[0]), "min_abs_sqrt_d": float(out[1]),
                "max_abs_sqrt_d": float(out[2]), "nonfinite": int(out[3])}

    def _gather(self, part):
        return self.comm.gather_partials(part)

    def forward(self) -> torch.Tensor:
        """Predicted data d (S*K_t*M_r,) on the device; stores g_i."""
        check(self.lib.rba_forward_partial(self.ctx, ptr(self.qpart)))
        self.g_valid = True
        d = torch.empty(self.S * self.Kt * self.Mr, dtype=torch.float64, device=self.device)
        if self.Mr == 0:
            return d
        qall = self._gather(self.qpart)
        check(self.lib.rba_combine_data(self.ctx, ptr(qall), ptr(self.slot_of_pole), 0, ptr(d)))
        return d

    def jvp(self, v: torch.Tensor) -> torch.Tensor:
        v = v.to(self.device, torch.float64).contiguous()
        check(self.lib.rba_jvp_partial(self.ctx, ptr(v), ptr(self.qpart)))
        qall = self._gather(self.qpart)
        d = torch.empty(self.S * self.Kt * self.Mr, dtype=torch.float64, device=self.device)
        check(self.lib.rba_combine_data(self.ctx, ptr(qall), ptr(self.slot_of_pole), 1, ptr(d)))
        return d

    def vjp(self, w: torch.Tensor) -> torch.Tensor:
        w = w.to(self.device, torch.float64).contiguous()
        check(self.lib.rba_vjp_partial(self.ctx, ptr(w), ptr(self.tpart)))
        tall = self._gather(self.tpart)
        out = torch.empty(self.P, dtype=torch.float64, device=self.device)
        check(self.lib.rba_combine_cells(self.ctx, ptr(tall), ptr(self.slot_of_pole), ptr(out)))
        return out

    # ------------------------------------------------------------ regulariser
    def set_reg(self, R: sp.spmatrix):
        R = sp.csr_matrix(R)
        R.sort_indices()
        if R.shape[1] != self.P:
            raise ValueError("regulariser must have P columns")
        self.reg_rows = R.shape[0]
        rp = np.ascontiguousarray(R.indptr, dtype=np.int64)
        ri = np.ascontiguousarray(R.indices, dtype=np.int32)
        rx = np.ascontiguousarray(R.data, dtype=np.float64)
        check(self.lib.rba_set_reg(self.ctx, R.shape[0], ptr(rp), ptr(ri), ptr(rx)))

    def set_reg_L(self, L: sp.spmatrix):
        L = sp.csr_matrix(L)
        L.sort_indices()
        if L.shape != (self.P, self.P):
            raise ValueError("L must be P x P")
        lp = np.ascontiguousarray(L.indptr, dtype=np.int64)
        li = np.ascontiguousarray(L.indices, dtype=np.int32)
        lx = np.ascontiguousarray(L.data, dtype=np.float64)
        check(self.lib.rba_set_reg_L(self.ctx, self.P, ptr(lp), ptr(li), ptr(lx)))

    def reg_L_apply(self, x: torch.Tensor, out: torch.Tensor, alpha=1.0, accumulate=False):
        check(self.lib.rba_reg_L_apply(self.ctx, ptr(x), float(alpha), ptr(out),
                                       1 if accumulate else 0))
        return out

    def reg_apply(self, x: torch.Tensor, out: torch.Tensor, alpha=1.0, transpose=False,
                  accumulate=False):
        check(self.lib.rba_reg_apply(self.ctx, 1 if transpose else 0, ptr(x), float(alpha),
                                     ptr(out), 1 if accumulate else 0))
        return out

    # ------------------------------------------------------------ vectors
    def axpby(self, a, x, b, y, out):
        check(self.lib.rba_vec_axpby(self.ctx, out.numel(), float(a), ptr(x), float(b),
                                     ptr(y if y is not None else x), ptr(out)))
        return out

    def mul(self, a, x, out, alpha=1.0):
        check(self.lib.rba_vec_mul(self.ctx, out.numel(), ptr(a), ptr(x), float(alpha), ptr(out)))
        return out

    def dot(self, x, y) -> float:
        r = _lib.f64()
        check(self.lib.rba_vec_dot(self.ctx, x.numel(), ptr(x), ptr(y), _lib.C.byref(r)))
        return r.value

    def lsqr_xw(self, t1, t2, v, w, x) -> float:
        r = _lib.f64()
        check(self.lib.rba_vec_lsqr_xw(self.ctx, x.numel(), float(t1), float(t2), ptr(v), ptr(w),
                                       ptr(x), _lib.C.byref(r)))
        return r.value

    # ------------------------------------------------------------ info
    def info(self) -> dict:
        out = np.zeros(10, np.int64)
        check(self.lib.rba_info(self.ctx, ptr(out)))
        mem = np.zeros(3, np.int64)
        check(self.lib.rba_memory(self.ctx, ptr(mem)))
        return dict(factorizations=int(out[0]), solves=int(out[1]), N=int(out[2]),
                    P=int(out[3]), Mr=int(out[4]), S=int(out[5]), m=int(out[6]),
                    n_local=int(out[7]), green=bool(out[8]), green_builds=int(out[9]),
                    mem_factor=int(mem[0]), mem_work=int(mem[1]),
                    mem_other=int(mem[2]))

    KCLASSES = ("scatter", "extend_add", "diag", "trsm", "gemm", "solve_fwd", "solve_bwd",
                "elem", "vec", "assembly", "green", "ozaki")

    def oz_stats(self) -> dict:
        """Ozaki-scheme INT8 Schur updates: on/off, int8 ops and FP64-equivalent
        flops per pole factorisation, poles per launch, pivot threshold."""
        out = np.zeros(5)
        check(self.lib.rba_oz_stats(self.ctx, ptr(out)))
        return {"on": bool(out[0]), "int8_ops_per_pole": float(out[1]),
                "flops_per_pole": float(out[2]), "poles_per_launch": int(out[3]),
                "min_pivots": int(out[4])}

    def oz_prof(self, reset: bool = True) -> dict:
        """Cycle counters of the Ozaki GEMM roles, summed over CTAs since the
        last reset (profiling aid, rba_oz_prof)."""
        out = np.zeros(10)
        check(self.lib.rba_oz_prof(self.ctx, ptr(out), 1 if reset else 0))
        keys = ("mma_loop", "mma_wait_data", "mma_wait_tmem", "producer_wait_stage",
                "epi_wait_acc", "epi_drain", "epi_rmw", "ksteps", "tiles", "mma_loop_ns")
        return dict(zip(keys, out.tolist()))

    def set_timing(self, mode):
        """True/1: record device time per kernel class; False/0: stop; 2: reset."""
        check(self.lib.rba_set_timing(self.ctx, int(mode)))

    def timings(self) -> dict:
        out = np.zeros(16)
        check(self.lib.rba_timings(self.ctx, ptr(out)))
        d = {k: float(out[i]) for i, k in enumerate(self.KCLASSES)}
        d["launches"] = int(out[15])
        return d

    def timings_detail(self) -> dict:
        out = np.zeros(128)
        check(self.lib.rba_timings_detail(self.ctx, ptr(out)))
        return {"solve_fwd_by_level": out[16:48].round(3).tolist(),
                "solve_bwd_by_level": out[48:80].round(3).tolist(),
                "factor_by_level": out[80:112].round(3).tolist(),
                "gemm_by_level": out[112:128].round(3).tolist()}

    def sync(self):
        check(self.lib.rba_sync(self.ctx))
