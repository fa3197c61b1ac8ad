"""Seeded synthetic inputs and the five BASELINE configurations.

BASELINE names no public dataset: these generators ARE the benchmark inputs.
  * counter-based uniform: x = splitmix64(seed ^ (stream << 40) ^ index),
    u = (x >> 11) * 2^-53, U[-1,1] = 2u - 1 -- bit-identical on host (numpy, here) and
    device (stkg_fill_uniform), so config 3's 8.6 GB F is generated in place on the GPU;
  * N(0,1) = Box-Muller on pairs of those uniforms (host only; small factor vectors):
    z_k uses u1 = 1 - u(2p), u2 = u(2p+1), p = k // 2, cos for even k, sin for odd k.
Streams: config * 16 + factor id.  Omega = (0,1)^d, I = (0,1), T = 1, zero initial and
boundary data; F is the already-projected load matrix, fed directly to the solver.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def uniform01(count: int, seed: int, stream: int, offset: int = 0) -> np.ndarray:
    idx = np.arange(offset, offset + count, dtype=np.uint64)
    key = np.uint64(seed) ^ (np.uint64(stream) << np.uint64(40))
    x = _splitmix64(key ^ idx)
    return (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_pm1(count: int, seed: int, stream: int, offset: int = 0) -> np.ndarray:
    return 2.0 * uniform01(count, seed, stream, offset) - 1.0


def normal(count: int, seed: int, stream: int) -> np.ndarray:
    pairs = (count + 1) // 2
    u = uniform01(2 * pairs, seed, stream)
    u1, u2 = 1.0 - u[0::2], u[1::2]
    r = np.sqrt(-2.0 * np.log(u1))
    z = np.empty(2 * pairs)
    z[0::2] = r * np.cos(2.0 * np.pi * u2)
    z[1::2] = r * np.sin(2.0 * np.pi * u2)
    return z[:count]


@dataclass(frozen=True)
class HeatConfig:
    name: str
    ndim: int
    n: int          # interior nodes per axis
    nt: int
    rank: int       # 0 = full-rank uniform F
    cid: int

    @property
    def nx(self) -> int:
        return self.n ** self.ndim

    @property
    def unknowns(self) -> int:
        return self.nx * self.nt


@dataclass(frozen=True)
class WaveConfig:
    name: str
    nh: int
    nt: int         # temporal elements (n_t + 1 cubic test functions)
    cid: int


CONFIGS = {
    "cfg1": HeatConfig("cfg1: 1D heat P1 255 x 256, rank-1 N(0,1) F", 1, 255, 256, 1, 1),
    "cfg2": HeatConfig("cfg2: 2D heat Q1 255^2 x 512, rank-4 N(0,1) F", 2, 255, 512, 4, 2),
    "cfg3": HeatConfig("cfg3: 2D heat Q1 1023^2 x 1024, full-rank U[-1,1] F", 2, 1023, 1024, 0, 3),
    "cfg4": WaveConfig("cfg4: 1D wave cubic splines 1023 x 1025, N(0,1) F", 1023, 1024, 4),
    "cfg5": HeatConfig("cfg5: 3D heat Q1 127^3 x 256, rank-8 N(0,1) F", 3, 127, 256, 8, 5),
}


def heat_factors(cfg: HeatConfig, seed: int = 0):
    """Low-rank factors (left n_x x r, right n_t x r) for rank>0 configs."""
    left = np.stack([normal(cfg.nx, seed, cfg.cid * 16 + 2 * r) for r in range(cfg.rank)], 1)
    right = np.stack([normal(cfg.nt, seed, cfg.cid * 16 + 2 * r + 1) for r in range(cfg.rank)], 1)
    return left, right


def heat_rhs_host(cfg: HeatConfig, seed: int = 0, nsteps: int | None = None) -> np.ndarray:
    """F as an (nsteps, n_x) C-order array == N_h x N_t column-major (first nsteps columns)."""
    nt = cfg.nt if nsteps is None else nsteps
    if cfg.rank == 0:
        return uniform_pm1(cfg.nx * nt, seed, cfg.cid * 16).reshape(nt, cfg.nx)
    left, right = heat_factors(cfg, seed)
    return np.ascontiguousarray(right[:nt] @ left.T)


def heat_rhs_host_slices(cfg: HeatConfig, j0: int, j1: int, seed: int = 0) -> np.ndarray:
    """Time slices j0..j1-1 of F (rows of the (n_t, n_x) C-order array), generated directly
    (the counter generator is random-access), for streaming a full-size solve on the host."""
    if cfg.rank == 0:
        return uniform_pm1(cfg.nx * (j1 - j0), seed, cfg.cid * 16,
                           offset=cfg.nx * j0).reshape(j1 - j0, cfg.nx)
    left, right = heat_factors(cfg, seed)
    return np.ascontiguousarray(right[j0:j1] @ left.T)


def wave_rhs_host(cfg: WaveConfig, seed: int = 0) -> np.ndarray:
    ntb = cfg.nt + 1
    return normal(cfg.nh * ntb, seed, cfg.cid * 16).reshape(ntb, cfg.nh)


def heat_rhs_device(cfg: HeatConfig, seed: int = 0, out=None):
    """F on the device.  Full-rank: generated in place by stkg_fill_uniform (bit-identical to
    heat_rhs_host); low-rank: factors built on the host, product formed on the device."""
    import ctypes as C

    import torch

    from ._lib import lib
    from .errors import check
    F = out if out is not None else torch.empty((cfg.nt, cfg.nx), dtype=torch.float64,
                                                device="cuda")
    if cfg.rank == 0:
        check(lib.stkg_fill_uniform(C.c_void_p(F.data_ptr()), F.numel(), seed, cfg.cid * 16, 0,
                                    C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    else:
        left, right = heat_factors(cfg, seed)
        L = torch.from_numpy(left).cuda()
        R = torch.from_numpy(right).cuda()
        torch.matmul(R, L.T, out=F)
    return F
