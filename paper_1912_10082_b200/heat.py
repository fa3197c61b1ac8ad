"""Heat hot path: the Python mirror of solve_projected_heat_with / KronOp over the C ABI.

Reference interface (stk/sylvester.hpp):
  * ``solve_projected_heat_with(eig, d, c, g)``  :117-142
  * ``heat_kron_op(m_h, a_h, d, c)`` / ``KronOp.apply(x)``  :58-65, :32-38
  * ``residual`` = ||F - KronOp.apply(U)||_F / ||F||_F  (stk/bench.hpp:508,524)

Layout: U and F are N_h x N_t column-major (space fastest), i.e. a contiguous buffer of
N_h * N_t doubles; as torch/numpy arrays that is shape (N_t, N_h) in C order.  The tensor
spatial index is ix*ny + iy (+ z fastest in 3D), the order of sparse_kron.

Device tensors (torch.float64 on CUDA) go through ``stkg_heat_solve``; host numpy arrays
go through ``stkg_heat_solve_host`` (H2D / solve / D2H pipelined over time chunks).
"""
from __future__ import annotations

import contextlib
import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from ._lib import HeatDesc, Report, RksmOpts, lib
from .assembly import Bidiagonal, EigPair, Tridiagonal
from .errors import ArgumentError, check

_dp = C.POINTER(C.c_double)


def _np_ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _dev_ptr(t) -> int:
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64):
        raise ArgumentError("expected a torch.float64 CUDA tensor")
    if not t.is_contiguous():
        raise ArgumentError("expected a contiguous tensor")
    return t.data_ptr()


@contextlib.contextmanager
def on_plan_stream(handle):
    """Order a plan call with the caller's current torch stream: the plan's stream waits
    for work already queued on the caller's stream (inputs written there), and the caller's
    stream waits for the plan's work (outputs used there).  A no-op when they are the same
    stream.  Plans bind their stream at creation; this keeps later calls made under another
    torch stream correct."""
    import torch
    if not torch.cuda.is_available():
        yield
        return
    cur = torch.cuda.current_stream()
    ph = int(handle.value or 0) if isinstance(handle, C.c_void_p) else int(handle or 0)
    if cur.cuda_stream == ph:
        yield
        return
    plan_stream = torch.cuda.ExternalStream(ph) if ph else torch.cuda.default_stream()
    plan_stream.wait_stream(cur)
    try:
        yield
    finally:
        cur.wait_stream(plan_stream)


def _stream_handle(stream):
    if stream is None:
        import torch
        if torch.cuda.is_available():
            return C.c_void_p(torch.cuda.current_stream().cuda_stream)
        return C.c_void_p(0)
    return C.c_void_p(int(stream))


@dataclass
class TensorEigPair:
    """EigPair of the Kronecker pencil: X = X_x (x) X_y (x) X_z, lambda = l_x (+) l_y (+) l_z."""
    axes: Sequence[EigPair]

    @property
    def shape(self):
        return tuple(int(e.lambdas.size) for e in self.axes)


class HeatPlan:
    """Prepared heat system on the GPU: tensor EigPair + temporal bidiagonals (+ the 1D
    spatial tridiagonals that define KronOp for apply/residual)."""

    def __init__(self, eig: TensorEigPair | EigPair, d: Bidiagonal, c: Bidiagonal,
                 m_axes: Sequence[Tridiagonal] | None = None,
                 a_axes: Sequence[Tridiagonal] | None = None, stream=None, time_chunk: int = 0,
                 transform: str = "dense", p1_h: Sequence[float] | None = None):
        """transform="dense": the per-axis X are applied as DMMA GEMMs (any EigPair).
        transform="dst": the axes carry the closed-form uniform-P1 eigenbasis of a grid of
        spacing p1_h[a] (X is not read) and are applied as FP64 fast sine transforms."""
        if isinstance(eig, EigPair):
            eig = TensorEigPair([eig])
        axes = list(eig.axes)
        ndim = len(axes)
        if not 1 <= ndim <= 3:
            raise ArgumentError("HeatPlan: 1 to 3 spatial axes")
        self.n = [int(e.lambdas.size) for e in axes]
        self.nt = int(d.diag.size)
        if c.diag.size != self.nt:
            raise ArgumentError("solve_projected_heat: D and C sizes differ")
        self.nx = int(np.prod(self.n))
        keep = []  # host arrays must outlive the create call

        def arr(a):
            a = np.ascontiguousarray(a, dtype=np.float64)
            keep.append(a)
            return _np_ptr(a)

        desc = HeatDesc()
        desc.ndim = ndim
        for i in range(3):
            desc.n[i] = self.n[i] if i < ndim else 1
        desc.nt = self.nt
        desc.d_diag, desc.c_diag = arr(d.diag), arr(c.diag)
        desc.d_sup = arr(d.sup if d.sup.size else np.zeros(1))
        desc.c_sup = arr(c.sup if c.sup.size else np.zeros(1))
        if transform not in ("dense", "dst"):
            raise ArgumentError("HeatPlan: transform must be 'dense' or 'dst'")
        desc.transform = 1 if transform == "dst" else 0
        if transform == "dst":
            if p1_h is None or len(p1_h) != ndim:
                raise ArgumentError("HeatPlan: transform='dst' needs p1_h per axis")
            for i in range(ndim):
                desc.p1_h[i] = float(p1_h[i])
        self.transform = transform
        for i, e in enumerate(axes):
            if transform == "dense":
                X = np.asfortranarray(e.X, dtype=np.float64)
                if X.shape != (self.n[i], self.n[i]):
                    raise ArgumentError("solve_projected_heat: EigPair X shape mismatch")
                keep.append(X)
                desc.X[i] = _np_ptr(X)
            desc.lambdas[i] = arr(e.lambdas)
        if m_axes is not None and a_axes is not None:
            for i in range(ndim):
                desc.m_diag[i] = arr(m_axes[i].diag)
                desc.m_off[i] = arr(m_axes[i].off if m_axes[i].off.size else np.zeros(1))
                desc.a_diag[i] = arr(a_axes[i].diag)
                desc.a_off[i] = arr(a_axes[i].off if a_axes[i].off.size else np.zeros(1))
        desc.time_chunk = int(time_chunk)
        self._stream = _stream_handle(stream)
        h = C.c_void_p()
        check(lib.stkg_heat_create(C.byref(h), C.byref(desc), self._stream))
        self._h = h

    @classmethod
    def p1_uniform(cls, ndim: int, n: int, nt: int, T: float = 1.0, a: float = 0.0,
                   b: float = 1.0, transform: str = "dst", with_operator: bool = True,
                   stream=None, time_chunk: int = 0) -> "HeatPlan":
        """Heat plan of the tensor P1/Q1 discretisation (fem1d_matrices per axis on (a,b) with
        n interior nodes, heat_time_matrices with nt steps on (0,T))."""
        from .assembly import SpaceGrid1D, TimeGrid, fem1d_matrices, heat_time_matrices, p1_eigpair
        g = SpaceGrid1D(a, b, n)
        M, A = fem1d_matrices(g)
        D, Cm = heat_time_matrices(TimeGrid(nt, T))
        e = p1_eigpair(g)
        ops = ([M] * ndim, [A] * ndim) if with_operator else (None, None)
        return cls(TensorEigPair([e] * ndim), D, Cm, ops[0], ops[1], stream=stream,
                   time_chunk=time_chunk, transform=transform, p1_h=[g.fem_h] * ndim)

    def close(self):
        if getattr(self, "_h", None):
            check(lib.stkg_heat_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def workspace_bytes(self) -> int:
        return int(lib.stkg_heat_workspace_bytes(self._h))

    def schedule(self) -> str:
        """The device schedule of :meth:`solve` (``stkg_heat_schedule``): ``"separate"`` (one
        transform pass per axis each way + the recurrence kernel), ``"fused_dst"`` (time-marching
        fused axis-0 pass) or ``"line_solve"`` (axis 0 solved by Toeplitz tridiagonal line solves,
        not transformed)."""
        return ("separate", "fused_dst", "line_solve")[int(lib.stkg_heat_schedule(self._h))]

    def _check_size(self, t):
        n = t.numel() if hasattr(t, "numel") else t.size
        if n != self.nx * self.nt:
            raise ArgumentError("solve_projected_heat: G shape mismatch")

    # -- device path ----------------------------------------------------------------
    def solve(self, F, out=None):
        """U = solve_projected_heat_with(eig, d, c, F) on device tensors."""
        import torch
        self._check_size(F)
        U = torch.empty_like(F) if out is None else out
        self._check_size(U)
        with on_plan_stream(self._stream):
            check(lib.stkg_heat_solve(self._h, C.c_void_p(_dev_ptr(F)), C.c_void_p(_dev_ptr(U))))
        return U

    def solve_factored(self, L, R, out=None):
        """Solve with a factored load F = L R^T (L: (rank, n_x) C-order == n_x x rank
        column-major, R: (rank, n_t)); F is never formed."""
        import torch
        rank = L.numel() // self.nx
        if L.numel() != rank * self.nx or R.numel() != rank * self.nt:
            raise ArgumentError("solve_factored: factor shape mismatch")
        U = torch.empty((self.nt, self.nx), dtype=torch.float64, device=L.device) if out is None else out
        self._check_size(U)
        with on_plan_stream(self._stream):
            check(lib.stkg_heat_solve_factored(self._h, rank, C.c_void_p(_dev_ptr(L)),
                                               C.c_void_p(_dev_ptr(R)), C.c_void_p(_dev_ptr(U))))
        return U

    def rksm(self, L, R, tol: float = 1e-8, maxit: int = 100, fixed_iters: int = 0,
             trunc_tol: float = 1e-10, cap: int | None = None):
        """rksm_solve (stk/rksm.hpp:127-234) for the load F = L R^T (L: (rank, n_x) C-order ==
        n_x x rank column-major, R: (rank, n_t)).  Returns (U_left (rank_u, n_x),
        U_right (rank_u, n_t), SolveReport) with U = U_left^T-stacked factors, i.e.
        U (n_t, n_x) C-order == U_right^T @ U_left."""
        import torch
        from .wave import _report
        rank = L.numel() // self.nx
        if L.numel() != rank * self.nx or R.numel() != rank * self.nt:
            raise ArgumentError("rksm_solve: F shape mismatch")
        cap = cap or max(1, min(self.nx, self.nt, rank * (maxit + 1)))
        UL = torch.empty((cap, self.nx), dtype=torch.float64, device=L.device)
        UR = torch.empty((cap, self.nt), dtype=torch.float64, device=L.device)
        opts = RksmOpts(tol, maxit, fixed_iters, trunc_tol)
        hist = np.zeros(max(maxit, fixed_iters) + 1)
        rep = Report()
        rep.rel_res_history = _np_ptr(hist)
        rep.history_capacity = hist.size
        rk = C.c_int64()
        with on_plan_stream(self._stream):
            check(lib.stkg_heat_rksm(self._h, rank, C.c_void_p(_dev_ptr(L)),
                                     C.c_void_p(_dev_ptr(R)), C.byref(opts),
                                     C.c_void_p(_dev_ptr(UL)), C.c_void_p(_dev_ptr(UR)), cap,
                                     C.byref(rk), C.byref(rep)))
        out = _report(rep, hist)
        out.rank = int(rk.value)
        return UL[: rk.value], UR[: rk.value], out

    def apply(self, U, out=None):
        """KronOp::apply of heat_kron_op: M U D + A U C."""
        import torch
        self._check_size(U)
        Y = torch.empty_like(U) if out is None else out
        self._check_size(Y)
        with on_plan_stream(self._stream):
            check(lib.stkg_heat_apply(self._h, C.c_void_p(_dev_ptr(U)), C.c_void_p(_dev_ptr(Y))))
        return Y

    def residual(self, U, F):
        """(||F - B(U)||_F / ||F||_F, ||F||_F), deterministic GPU reduction (K1)."""
        self._check_size(U)
        self._check_size(F)
        rel, fn = C.c_double(), C.c_double()
        with on_plan_stream(self._stream):
            check(lib.stkg_heat_residual(self._h, C.c_void_p(_dev_ptr(U)),
                                         C.c_void_p(_dev_ptr(F)), C.byref(rel), C.byref(fn)))
        return rel.value, fn.value

    # -- profiling ------------------------------------------------------------------
    def profile_begin(self):
        check(lib.stkg_heat_profile(self._h, 1, None, None))

    def profile_end(self):
        """-> {"transform": (ms, launches), "scan": (ms, launches)} since profile_begin:
        class "transform" = transform-only passes, "scan" = kernels that run the modal
        recurrence (the scan kernel, or the fused axis-0 pass)."""
        ms = (C.c_double * 2)()
        n = (C.c_int64 * 2)()
        check(lib.stkg_heat_profile(self._h, 0, ms, n))
        return {"transform": (ms[0], n[0]), "scan": (ms[1], n[1])}

    # -- host path ------------------------------------------------------------------
    def solve_host(self, F: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """Same solve with host buffers; H2D, solve and D2H overlap across time chunks."""
        F = np.ascontiguousarray(F, dtype=np.float64)
        self._check_size(F)
        U = np.empty_like(F) if out is None else out
        if not (isinstance(U, np.ndarray) and U.flags.c_contiguous and U.dtype == np.float64
                and U.flags.writeable):
            raise ArgumentError("solve_host: out must be a writable contiguous float64 array")
        self._check_size(U)  # the D2H copy writes n_x * n_t doubles
        check(lib.stkg_heat_solve_host(self._h, C.c_void_p(F.ctypes.data),
                                       C.c_void_p(U.ctypes.data)))
        return U


def solve_projected_heat_with(eig, d: Bidiagonal, c: Bidiagonal, g):
    """Reference-named entry point (stk/sylvester.hpp:117): one-shot plan + solve.

    ``g`` may be a device tensor (result on device) or a host numpy array (result on host).
    """
    plan = HeatPlan(eig, d, c)
    try:
        if isinstance(g, np.ndarray):
            return plan.solve_host(g)
        return plan.solve(g)
    finally:
        plan.close()


class HeatKronOp:
    """heat_kron_op(M, A, D, C) (stk/sylvester.hpp:58-65) for tensor-grid Q1/P1 factors:
    M = (x) M_axis, A = sum_axis A_axis (x) M_others (fem2d_matrices, :81-88)."""

    def __init__(self, m_axes: Sequence[Tridiagonal], a_axes: Sequence[Tridiagonal],
                 d: Bidiagonal, c: Bidiagonal, eig: TensorEigPair | None = None, stream=None):
        if eig is None:  # apply-only plan: identity eigen-data is never used by apply
            eig = TensorEigPair([EigPair(np.ones(m.diag.size), np.eye(m.diag.size))
                                 for m in m_axes])
        self.plan = HeatPlan(eig, d, c, m_axes, a_axes, stream=stream)

    def apply(self, U, out=None):
        return self.plan.apply(U, out)


def heat_kron_op(m_axes, a_axes, d, c, eig=None):
    return HeatKronOp(m_axes, a_axes, d, c, eig)
