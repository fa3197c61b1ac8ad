"""B200-native (sm_100a, FP64) Kronecker space-time solver: the hot path of stk
(arXiv:1912.10082) behind the reference's own entry points.

The compute path is the CUDA library ``_stk_gpu.so`` (include/stk_gpu.h); importing this
package loads it (building it in-tree with nvcc if needed) and fails loudly otherwise.
There is no CPU fallback.
"""
from . import _lib  # noqa: F401  (loads the CUDA library or raises)
from .assembly import (Band7, Bidiagonal, EigPair, SpaceGrid1D, TimeGrid, Tridiagonal,
                       WaveSpaceMatrices, WaveTimeMatrices, fem1d_matrices, heat_time_matrices,
                       p1_eigpair, sym_gen_eig, wave_space_matrices, wave_time_dim,
                       wave_time_matrices)
from .errors import (ArgumentError, CudaError, DefinitenessError, NumericError,
                     SingularityError, SolvabilityError, StkError)
from .heat import HeatKronOp, HeatPlan, TensorEigPair, heat_kron_op, solve_projected_heat_with
from .wave import (GmresConfig, SolveReport, TwoTermPrecond, WaveOperator, WavePlan, gmres)
from . import formats  # noqa: E402
from .formats import ResultRow, read_matrix_market, write_history_csv, write_matrix_market

__all__ = [n for n in dir() if not n.startswith("_")]
