"""Host-side assembly (layer L1): Python view of the C ABI's host entry points.

Mirrors stk/discretize.hpp (TimeGrid, SpaceGrid1D, heat_time_matrices, fem1d_matrices,
wave_time_matrices, wave_space_matrices) and stk/la_core.hpp:64-91 (sym_gen_eig).  All
arrays are numpy float64; band matrices use the layout of include/stk_gpu.h
(band[d, i] = Mat[i, i + d - 3]).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import lib
from .errors import ArgumentError, check


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


@dataclass(frozen=True)
class TimeGrid:
    """Uniform temporal grid with nt elements on (0, T) (stk/discretize.hpp:13-24)."""
    nt: int
    T: float = 1.0

    def __post_init__(self):
        if self.nt < 1:
            raise ArgumentError("TimeGrid: nt must be >= 1")
        if not self.T > 0:
            raise ArgumentError("TimeGrid: T must be positive")

    @property
    def dt(self) -> float:
        return self.T / self.nt


@dataclass(frozen=True)
class SpaceGrid1D:
    """1D interval (a, b) with nh active functions (stk/discretize.hpp:28-39)."""
    a: float
    b: float
    nh: int

    def __post_init__(self):
        if not self.b > self.a:
            raise ArgumentError("SpaceGrid1D: empty interval")
        if self.nh < 1:
            raise ArgumentError("SpaceGrid1D: nh must be >= 1")

    @property
    def fem_h(self) -> float:
        return (self.b - self.a) / (self.nh + 1)


@dataclass
class Bidiagonal:
    """Upper bidiagonal n x n matrix: diag (n), sup (n-1; sup[k] = [k, k+1])."""
    diag: np.ndarray
    sup: np.ndarray

    def dense(self) -> np.ndarray:
        n = self.diag.size
        m = np.diag(self.diag)
        if n > 1:
            m += np.diag(self.sup, 1)
        return m


@dataclass
class Tridiagonal:
    """Symmetric tridiagonal n x n matrix: diag (n), off (n-1)."""
    diag: np.ndarray
    off: np.ndarray

    def dense(self) -> np.ndarray:
        m = np.diag(self.diag)
        if self.diag.size > 1:
            m += np.diag(self.off, 1) + np.diag(self.off, -1)
        return m


@dataclass
class Band7:
    """7-diagonal n x n matrix, band[d, i] = A[i, i + d - 3]."""
    band: np.ndarray  # (7, n)

    @property
    def n(self) -> int:
        return self.band.shape[1]

    def dense(self) -> np.ndarray:
        n = self.n
        m = np.zeros((n, n))
        for d in range(7):
            for i in range(n):
                j = i + d - 3
                if 0 <= j < n:
                    m[i, j] = self.band[d, i]
        return m


@dataclass
class EigPair:
    """Generalized eigenpair Q X = M X diag(lambdas), X^T M X = I (stk/types.hpp:126-129)."""
    lambdas: np.ndarray
    X: np.ndarray  # n x n (numpy array; column k = eigenvector k)


def heat_time_matrices(grid: TimeGrid):
    """(D, C) upper bidiagonal (stk/discretize.hpp:44-57)."""
    n = grid.nt
    dd, cd = np.empty(n), np.empty(n)
    ds, cs = np.empty(max(n - 1, 1)), np.empty(max(n - 1, 1))
    check(lib.stkg_heat_time_matrices(n, grid.T, _p(dd), _p(ds), _p(cd), _p(cs)))
    return Bidiagonal(dd, ds[: n - 1].copy()), Bidiagonal(cd, cs[: n - 1].copy())


def fem1d_matrices(grid: SpaceGrid1D):
    """(M_h, A_h) P1 mass/stiffness (stk/discretize.hpp:61-77)."""
    n = grid.nh
    md, ad = np.empty(n), np.empty(n)
    mo, ao = np.empty(max(n - 1, 1)), np.empty(max(n - 1, 1))
    check(lib.stkg_fem1d_matrices(grid.a, grid.b, n, _p(md), _p(mo), _p(ad), _p(ao)))
    return Tridiagonal(md, mo[: n - 1].copy()), Tridiagonal(ad, ao[: n - 1].copy())


def p1_eigpair(grid: SpaceGrid1D) -> EigPair:
    """Closed-form sym_gen_eig(A_h, M_h) for the uniform P1 pencil."""
    n = grid.nh
    X = np.empty((n, n), order="F")
    lam = np.empty(n)
    check(lib.stkg_p1_eigpair(grid.a, grid.b, n, _p(X), _p(lam)))
    return EigPair(lam, X)


def sym_gen_eig(Q: np.ndarray, M: np.ndarray) -> EigPair:
    """Generalized symmetric-definite eigenproblem (stk/la_core.hpp:64-91), host C++."""
    Q = np.asfortranarray(Q, dtype=np.float64)
    M = np.asfortranarray(M, dtype=np.float64)
    n = Q.shape[0]
    if Q.shape != (n, n) or M.shape != (n, n):
        raise ArgumentError("sym_gen_eig: size mismatch")
    X = np.empty((n, n), order="F")
    lam = np.empty(n)
    check(lib.stkg_sym_gen_eig(n, _p(Q), _p(M), _p(lam), _p(X)))
    return EigPair(lam, X)


@dataclass
class WaveSpaceMatrices:
    M: Band7  # (psi_i, psi_j)
    A: Band7  # (psi_i', psi_j')
    Q: Band7  # (psi_i'', psi_j'')


@dataclass
class WaveTimeMatrices:
    Q: Band7  # (rho_ddot^k, rho_ddot^l)
    D: Band7  # (rho_ddot^k, rho^l)
    M: Band7  # (rho^k, rho^l)


def wave_space_matrices(grid: SpaceGrid1D, degree: int = 3) -> WaveSpaceMatrices:
    """stk/discretize.hpp:154-161 on wave_space_basis(grid, degree) (:99-104)."""
    n = grid.nh
    bands = np.zeros(3 * 7 * n)
    check(lib.stkg_wave_space_matrices(grid.a, grid.b, n, degree, _p(bands)))
    b = bands.reshape(3, 7, n)
    return WaveSpaceMatrices(Band7(b[0].copy()), Band7(b[1].copy()), Band7(b[2].copy()))


def wave_time_dim(nt: int, degree: int = 3) -> int:
    return int(lib.stkg_wave_time_dim(nt, degree))


def wave_time_matrices(grid: TimeGrid, degree: int = 3) -> WaveTimeMatrices:
    """stk/discretize.hpp:141-146 on wave_time_basis(grid, degree) (:92-95)."""
    n = wave_time_dim(grid.nt, degree)
    bands = np.zeros(3 * 7 * n)
    check(lib.stkg_wave_time_matrices(grid.nt, grid.T, degree, _p(bands)))
    b = bands.reshape(3, 7, n)
    return WaveTimeMatrices(Band7(b[0].copy()), Band7(b[1].copy()), Band7(b[2].copy()))
