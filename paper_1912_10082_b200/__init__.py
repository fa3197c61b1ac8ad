"""B200-native (sm_100a, FP64) Kronecker space-time solver: the hot path of stk
(arXiv:1912.10082) behind the reference's own entry points.

The compute path is the CUDA library ``_stk_gpu.so`` (include/stk_gpu.h).  It is loaded
(built in-tree with nvcc if needed) the first time any solver, assembly or error symbol of
this package is touched, and that access raises if the library cannot be loaded: there is
no CPU fallback.  The host-only modules ``inputs`` (seeded synthetic inputs) and
``formats`` (CSV / MatrixMarket) do not map the library, so a CPU-only process -- the
bench's reference arm -- can generate the same inputs without loading any CUDA code.
"""
from __future__ import annotations

import importlib

_EXPORTS = {
    ".assembly": ("Band7", "Bidiagonal", "EigPair", "SpaceGrid1D", "TimeGrid", "Tridiagonal",
                  "WaveSpaceMatrices", "WaveTimeMatrices", "fem1d_matrices",
                  "heat_time_matrices", "p1_eigpair", "sym_gen_eig", "wave_space_matrices",
                  "wave_time_dim", "wave_time_matrices"),
    ".errors": ("ArgumentError", "CudaError", "DefinitenessError", "NumericError",
                "SingularityError", "SolvabilityError", "StkError"),
    ".heat": ("HeatKronOp", "HeatPlan", "TensorEigPair", "heat_kron_op",
              "solve_projected_heat_with"),
    ".wave": ("GmresConfig", "SolveReport", "TwoTermPrecond", "WaveOperator", "WavePlan",
              "gmres"),
    ".formats": ("ResultRow", "read_matrix_market", "write_history_csv",
                 "write_matrix_market"),
}
_WHERE = {name: mod for mod, names in _EXPORTS.items() for name in names}
_LIB_FREE = {".formats"}  # host-only modules that never touch the CUDA library

__all__ = sorted(_WHERE) + ["formats", "inputs"]


def __getattr__(name: str):
    mod = _WHERE.get(name)
    if mod is None:
        if name in ("formats", "inputs", "heat", "wave", "assembly", "errors"):
            return importlib.import_module("." + name, __name__)
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    if mod not in _LIB_FREE:
        importlib.import_module("._lib", __name__)  # loads the CUDA library or raises
    value = getattr(importlib.import_module(mod, __name__), name)
    globals()[name] = value
    return value


def __dir__():
    return __all__
