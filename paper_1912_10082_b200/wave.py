"""Wave hot path: Python mirror of WaveOperator / TwoTermPrecond / gmres over the C ABI.

Reference interface:
  * ``WaveOperator(m_h, a_h, q_h, q_dt, d_dt, m_dt).apply(x)``  stk/outer_krylov.hpp:168-191
  * ``TwoTermPrecond(m_h, q_h, m_dt, q_dt).solve(v)``          stk/sylvester.hpp:153-181
  * ``gmres(apply, precond, b, cfg) -> (x, SolveReport)``      stk/outer_krylov.hpp:75-164
  * ``GmresConfig`` (:18-28), ``SolveReport`` (stk/report.hpp:11-20)

``gmres`` takes either the plan objects (apply = WaveOperator, precond = TwoTermPrecond, the
pairing run_wave_experiment passes through the VecOp seam, stk/bench.hpp:667-673; both
live in one device plan) or arbitrary callables on device vectors (``stkg_gmres_op``).
``pcg`` is the s.p.d. performance path.
"""
from __future__ import annotations

import contextlib
import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import VEC_OP, GmresCfg, Report, WaveDesc, lib
from .assembly import EigPair, WaveSpaceMatrices, WaveTimeMatrices, sym_gen_eig
from .errors import ArgumentError, check
from .heat import _dev_ptr, _np_ptr, _stream_handle, on_plan_stream


@dataclass
class GmresConfig:
    tol: float = 1e-8
    maxit: int = 200
    restart: int = 0  # 0 = full GMRES

    def validate(self):
        if not 0.0 < self.tol < 1.0:
            raise ArgumentError("GmresConfig: tol must be in (0,1)")
        if self.maxit < 1:
            raise ArgumentError("GmresConfig: maxit must be >= 1")


@dataclass
class SolveReport:
    iterations: int = 0
    rel_res_history: list = field(default_factory=list)
    mu_mem: int = 0
    rank: int = 0
    wall_time_s: float = 0.0
    final_relres: float = 0.0
    converged: bool = False
    stagnated: bool = False


def _report(r: Report, hist: np.ndarray) -> SolveReport:
    n = min(r.history_length, hist.size)
    return SolveReport(iterations=r.iterations, rel_res_history=hist[:n].tolist(),
                       mu_mem=r.mu_mem, wall_time_s=r.wall_time_s, final_relres=r.final_relres,
                       converged=bool(r.converged), stagnated=bool(r.stagnated))


class WavePlan:
    """Device plan of the wave system: the six banded factors and (optionally) the two
    generalized eigenpairs of TwoTermPrecond."""

    PRECONDS = {"two_term": 0, "modal_banded": 1}

    def __init__(self, space: WaveSpaceMatrices, time: WaveTimeMatrices, precond: bool = True,
                 space_eig: EigPair | None = None, time_eig: EigPair | None = None, stream=None,
                 preconditioner: str = "two_term"):
        """preconditioner: what gmres / pcg / solve_refined apply -- "two_term" (the
        reference's TwoTermPrecond, default) or "modal_banded" (stkg_modal_banded_solve:
        A_h diagonalised in the same eigenbasis, a banded s.p.d. time solve per spatial
        mode; ~10 PCG iterations at every size)."""
        if preconditioner not in self.PRECONDS:
            raise ArgumentError(f"WavePlan: unknown preconditioner {preconditioner!r}")
        self.nh = space.M.n
        self.nt = time.M.n
        keep = []

        def arr(a):
            a = np.ascontiguousarray(a, dtype=np.float64)
            keep.append(a)
            return _np_ptr(a)

        desc = WaveDesc()
        desc.nh, desc.nt = self.nh, self.nt
        desc.space_bands = arr(np.concatenate([space.M.band, space.A.band, space.Q.band]))
        desc.time_bands = arr(np.concatenate([time.Q.band, time.D.band, time.M.band]))
        self.space_eig = self.time_eig = None
        if precond:
            # TwoTermPrecond ctor (stk/sylvester.hpp:155-161): sym_gen_eig(Q_h, M_h), (Q_t, M_t)
            self.space_eig = space_eig or sym_gen_eig(space.Q.dense(), space.M.dense())
            self.time_eig = time_eig or sym_gen_eig(time.Q.dense(), time.M.dense())
            Xs = np.asfortranarray(self.space_eig.X)
            Xt = np.asfortranarray(self.time_eig.X)
            keep += [Xs, Xt]
            desc.Xs, desc.Xt = _np_ptr(Xs), _np_ptr(Xt)
            desc.lambdas = arr(self.space_eig.lambdas)
            desc.thetas = arr(self.time_eig.lambdas)
        h = C.c_void_p()
        self._stream = _stream_handle(stream)
        check(lib.stkg_wave_create(C.byref(h), C.byref(desc), self._stream))
        self._h = h
        self.preconditioner = "two_term"
        if precond:
            self.set_preconditioner(preconditioner)

    def set_preconditioner(self, name: str):
        if name not in self.PRECONDS:
            raise ArgumentError(f"WavePlan: unknown preconditioner {name!r}")
        check(lib.stkg_wave_set_precond(self._h, self.PRECONDS[name]))
        self.preconditioner = name

    def close(self):
        if getattr(self, "_h", None):
            check(lib.stkg_wave_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def N(self):
        return self.nh * self.nt

    def _chk(self, t):
        if t.numel() != self.N:
            raise ArgumentError("WaveOperator: vector length mismatch")

    def apply(self, x, out=None):
        import torch
        self._chk(x)
        y = torch.empty_like(x) if out is None else out
        self._chk(y)
        with on_plan_stream(self._stream):
            check(lib.stkg_wave_apply(self._h, C.c_void_p(_dev_ptr(x)), C.c_void_p(_dev_ptr(y))))
        return y

    def modal_banded_solve(self, v, out=None):
        """P^-1 v for the space-modal time-banded preconditioner (stkg_modal_banded_solve)."""
        import torch
        self._chk(v)
        w = torch.empty_like(v) if out is None else out
        self._chk(w)
        with on_plan_stream(self._stream):
            check(lib.stkg_modal_banded_solve(self._h, C.c_void_p(_dev_ptr(v)),
                                              C.c_void_p(_dev_ptr(w))))
        return w

    def two_term_solve(self, v, out=None):
        import torch
        self._chk(v)
        w = torch.empty_like(v) if out is None else out
        self._chk(w)
        with on_plan_stream(self._stream):
            check(lib.stkg_two_term_solve(self._h, C.c_void_p(_dev_ptr(v)),
                                          C.c_void_p(_dev_ptr(w))))
        return w

    def gmres(self, b, cfg: GmresConfig | None = None, precond: bool = True, x=None):
        import torch
        cfg = cfg or GmresConfig()
        cfg.validate()
        self._chk(b)
        x = torch.empty_like(b) if x is None else x
        self._chk(x)
        c = GmresCfg(cfg.tol, cfg.maxit, cfg.restart, 1 if precond else 0)
        hist = np.zeros(cfg.maxit + 1)
        rep = Report()
        rep.rel_res_history = _np_ptr(hist)
        rep.history_capacity = hist.size
        with on_plan_stream(self._stream):
            check(lib.stkg_gmres(self._h, C.c_void_p(_dev_ptr(b)), C.c_void_p(_dev_ptr(x)),
                                 C.byref(c), C.byref(rep)))
        return x, _report(rep, hist)

    def pcg(self, b, tol: float = 1e-8, maxit: int = 1000, x=None):
        import torch
        self._chk(b)
        x = torch.empty_like(b) if x is None else x
        self._chk(x)
        hist = np.zeros(maxit + 1)
        rep = Report()
        rep.rel_res_history = _np_ptr(hist)
        rep.history_capacity = hist.size
        with on_plan_stream(self._stream):
            check(lib.stkg_pcg(self._h, C.c_void_p(_dev_ptr(b)), C.c_void_p(_dev_ptr(x)), tol,
                               maxit, C.byref(rep)))
        return x, _report(rep, hist)

    def residual_dd(self, b, x_hi, x_lo=None, out=None) -> float:
        """||b - B (x_hi + x_lo)|| / ||b|| with the residual evaluated in double-double
        (stkg_wave_residual_dd); the FP64-rounded residual vector lands in out if given."""
        self._chk(b)
        self._chk(x_hi)
        for t in (x_lo, out):
            if t is not None:
                self._chk(t)
        rel = C.c_double()
        with on_plan_stream(self._stream):
            check(lib.stkg_wave_residual_dd(
                self._h, C.c_void_p(_dev_ptr(b)), C.c_void_p(_dev_ptr(x_hi)),
                C.c_void_p(_dev_ptr(x_lo) if x_lo is not None else None),
                C.c_void_p(_dev_ptr(out) if out is not None else None), C.byref(rel)))
        return rel.value

    def solve_refined(self, b, tol: float = 1e-10, max_refine: int = 6,
                      inner_tol: float = 1e-6, inner_maxit: int = 6000):
        """Mixed-precision iterative refinement (stkg_wave_solve_refined): returns
        (x_hi, x_lo, SolveReport) with the solution x_hi + x_lo as a double-double pair;
        rel_res_history holds the double-double relative residual per round."""
        import torch
        self._chk(b)
        xh = torch.empty_like(b)
        xl = torch.empty_like(b)
        hist = np.zeros(max_refine + 2)
        rep = Report()
        rep.rel_res_history = _np_ptr(hist)
        rep.history_capacity = hist.size
        with on_plan_stream(self._stream):
            check(lib.stkg_wave_solve_refined(self._h, C.c_void_p(_dev_ptr(b)),
                                              C.c_void_p(_dev_ptr(xh)), C.c_void_p(_dev_ptr(xl)),
                                              tol, max_refine, inner_tol, inner_maxit,
                                              C.byref(rep)))
        return xh, xl, _report(rep, hist)


class WaveOperator:
    """vec(M_h U Q_t^T + A_h U (D_t + D_t^T) + Q_h U M_t) (stk/outer_krylov.hpp:168-191)."""

    def __init__(self, plan: WavePlan):
        self.plan = plan

    def space_dim(self):
        return self.plan.nh

    def time_dim(self):
        return self.plan.nt

    def apply(self, x, out=None):
        return self.plan.apply(x, out)


class TwoTermPrecond:
    """M_h W Q_t^T + Q_h W M_t = V solved in the eigenbases (stk/sylvester.hpp:153-181)."""

    def __init__(self, plan: WavePlan):
        if plan.space_eig is None:
            raise ArgumentError("TwoTermPrecond: plan built without eigenpairs")
        self.plan = plan

    def space(self) -> EigPair:
        return self.plan.space_eig

    def time(self) -> EigPair:
        return self.plan.time_eig

    def solve(self, v, out=None):
        return self.plan.two_term_solve(v, out)


class _DevView:
    """Zero-copy torch view of a raw device vector (via __cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8",
                                         "data": (ptr, False), "version": 3, "strides": None}


def _vec_op(fn, n):
    import torch

    def cb(user, x, y, stream):
        try:
            xs = torch.as_tensor(_DevView(x, n), device="cuda")
            ys = torch.as_tensor(_DevView(y, n), device="cuda")
            ctx = (torch.cuda.stream(torch.cuda.ExternalStream(stream)) if stream
                   else contextlib.nullcontext())
            with ctx:
                out = fn(xs)
                if out is not None and out.data_ptr() != y:
                    ys.copy_(out.reshape(-1))
            return 0
        except ArgumentError:
            return 1
        except Exception:  # surfaced as NumericError by the solver
            return 5
    return VEC_OP(cb)


def gmres(apply, precond, b, cfg: GmresConfig | None = None):
    """gmres(apply, precond, b, cfg) -> (x, SolveReport) (stk/outer_krylov.hpp:75-164).

    ``apply``/``precond`` are either the plan objects (WaveOperator, TwoTermPrecond of one
    WavePlan: everything stays in the library) or arbitrary callables on torch CUDA vectors
    -- the reference's VecOp seam (:30), run through ``stkg_gmres_op``."""
    import torch
    cfg = cfg or GmresConfig()
    cfg.validate()
    if isinstance(apply, WaveOperator) and (precond is None or isinstance(precond, TwoTermPrecond)):
        if precond is not None and precond.plan is not apply.plan:
            raise ArgumentError("gmres: operator and preconditioner must share one WavePlan")
        return apply.plan.gmres(b, cfg, precond=precond is not None)
    fa = apply.apply if hasattr(apply, "apply") else apply
    fp = None if precond is None else (precond.solve if hasattr(precond, "solve") else precond)
    n = b.numel()
    x = torch.empty_like(b)
    cb_a = _vec_op(fa, n)
    cb_p = _vec_op(fp, n) if fp is not None else VEC_OP()
    c = GmresCfg(cfg.tol, cfg.maxit, cfg.restart, 1 if fp is not None else 0)
    hist = np.zeros(cfg.maxit + 1)
    rep = Report()
    rep.rel_res_history = _np_ptr(hist)
    rep.history_capacity = hist.size
    stream = torch.cuda.current_stream().cuda_stream
    check(lib.stkg_gmres_op(n, cb_a, None, cb_p, None, C.c_void_p(_dev_ptr(b)),
                            C.c_void_p(_dev_ptr(x)), C.byref(c), C.byref(rep), C.c_void_p(stream)))
    return x, _report(rep, hist)
