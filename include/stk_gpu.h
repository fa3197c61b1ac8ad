/*
 * stk_gpu.h -- C ABI of the B200-native (sm_100a, FP64) Kronecker space-time solver.
 *
 * This is the drop-in boundary for the hot path of the reference library `stk`
 * (/root/reference/proj/include/stk).  Every entry point below names the reference
 * function it replaces (file:line, paths relative to proj/include/).  No C++ or torch
 * types cross this boundary: plain pointers, 64-bit sizes, int status codes.
 *
 * Conventions (identical to the reference, stk/types.hpp, stk/outer_krylov.hpp:181):
 *   - all matrices are column-major FP64; U, F are N_h x N_t with space fastest and
 *     vec(U) = column stacking;
 *   - the tensor spatial index is ix*ny + iy (2D) and (ix*ny + iy)*nz + iz (3D),
 *     i.e. the order of sparse_kron (stk/types.hpp:131-145);
 *   - pointers documented "device" are CUDA device pointers, "host" are host pointers;
 *   - every call is asynchronous on the object's stream unless it returns a host value.
 *
 * Status codes map 1:1 onto the reference exception classes (stk/errors.hpp:9-42).
 * stkg_last_error_message() returns the message of the last failing call on the calling
 * thread (thread-local), the analogue of exception::what().
 */
#ifndef STK_GPU_H
#define STK_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  STKG_OK = 0,
  STKG_ARGUMENT = 1,      /* stk::ArgumentError      (stk/errors.hpp:9)  */
  STKG_DEFINITENESS = 2,  /* stk::DefinitenessError  (stk/errors.hpp:15) */
  STKG_SINGULARITY = 3,   /* stk::SingularityError   (stk/errors.hpp:21) */
  STKG_SOLVABILITY = 4,   /* stk::SolvabilityError   (stk/errors.hpp:27) */
  STKG_NUMERIC = 5,       /* stk::NumericError       (stk/errors.hpp:33) */
  STKG_CUDA = 6           /* CUDA runtime failure (no reference counterpart) */
};

const char* stkg_last_error_message(void);
const char* stkg_version(void);

/* ---------------------------------------------------------------- device memory --- */
/* Thin helpers so that a C / cgo / JNI caller needs no CUDA headers. */
int stkg_device_alloc(void** ptr, size_t bytes);
int stkg_device_free(void* ptr);
int stkg_memcpy_h2d(void* dst, const void* src, size_t bytes);
int stkg_memcpy_d2h(void* dst, const void* src, size_t bytes);
int stkg_device_synchronize(void);
/* Fill dst[0..count) with Uniform[-1,1) from the counter-based splitmix64 generator of
 * x = splitmix64(seed ^ (stream << 40) ^ index), u = (x >> 11) * 2^-53,
 * value = 2u - 1.  Bit-identical to the host generator (oracle and bench). */
int stkg_fill_uniform(double* dst_device, int64_t count, uint64_t seed, uint64_t stream,
                      int64_t index_offset, void* cuda_stream);

/* ------------------------------------------------------ host-side assembly (L1) --- */
/* These run on the host; they build the factors the GPU plans consume.               */

/* heat_time_matrices (stk/discretize.hpp:44-57): D, C upper bidiagonal, n_t x n_t.
 * d_diag/c_diag have nt entries, d_sup/c_sup nt-1 (entry k is [k, k+1]). */
int stkg_heat_time_matrices(int nt, double T, double* d_diag, double* d_sup,
                            double* c_diag, double* c_sup);
/* fem1d_matrices (stk/discretize.hpp:61-77): P1 mass/stiffness on (a,b), nh interior
 * nodes; symmetric tridiagonal, off arrays have nh-1 entries. */
int stkg_fem1d_matrices(double a, double b, int nh, double* m_diag, double* m_off,
                        double* a_diag, double* a_off);
/* Closed-form generalized eigenpair of the uniform P1 pencil (A_h, M_h) on (a,b)
 * (SURVEY Appendix A); replaces sym_gen_eig(A_h, M_h) (stk/la_core.hpp:64-91) for the
 * uniform grid.  X is nh x nh column-major, X^T M X = I, lambdas ascending. */
int stkg_p1_eigpair(double a, double b, int nh, double* X, double* lambdas);
/* sym_gen_eig (stk/la_core.hpp:64-91): Cholesky M = L L^T, eigen-decomposition of the
 * symmetrized L^-1 Q L^-T (Householder tridiagonalisation + implicit QL), X = L^-T V.
 * Q, M dense n x n column-major (host).  STKG_DEFINITENESS if M is not s.p.d. */
int stkg_sym_gen_eig(int n, const double* Q, const double* M, double* lambdas, double* X);
/* Wave spline Gram matrices as 7-diagonal bands (degree 3) -- band layout:
 * band[d * n + i] = Mat[i, i + d - 3], d = 0..6 (zero outside the matrix).
 * wave_space_matrices (stk/discretize.hpp:154-161) on (a,b) with nh active functions:
 *   out = [M | A | Q] (3 bands of 7*nh).  wave_time_matrices (stk/discretize.hpp:141-146)
 * on (0,T) with nt elements: n_tb = nt + degree - 2 active functions (wave_time_basis,
 *   stk/discretize.hpp:92-95), out = [Q | D | M] (3 bands of 7*n_tb).
 * Entries follow spline_gram (stk/discretize.hpp:111-131), summed in triplet order. */
int stkg_wave_space_matrices(double a, double b, int nh, int degree, double* bands);
int stkg_wave_time_dim(int nt, int degree);
int stkg_wave_time_matrices(int nt, double T, int degree, double* bands);

/* ------------------------------------------------------------------ heat plans --- */
/* A heat plan holds the data solve_projected_heat_with(eig, d, c, g)
 * (stk/sylvester.hpp:117-142) reads, for a tensor EigPair X = X_x (x) X_y (x) X_z,
 * lambda = lambda_x (+) lambda_y (+) lambda_z, plus the 1D
 * tridiagonal factors that define KronOp heat_kron_op(M, A, D, C)
 * (stk/sylvester.hpp:58-65) with M = (x) M_axis, A = sum_axis A_axis (x) M_others
 * (fem2d_matrices, stk/discretize.hpp:81-88). */
typedef struct stkg_heat stkg_heat;

typedef struct stkg_heat_desc {
  int ndim;                 /* 1, 2 or 3 */
  int64_t n[3];             /* interior nodes per axis, x slowest; n[1], n[2] unused below ndim */
  int64_t nt;               /* temporal dimension (columns of U) */
  const double* d_diag;     /* host, nt    -- upper bidiagonal D (heat_time_matrices) */
  const double* d_sup;      /* host, nt-1 */
  const double* c_diag;     /* host, nt    -- upper bidiagonal C */
  const double* c_sup;      /* host, nt-1 */
  const double* X[3];       /* host, n[a] x n[a] column-major per-axis eigenvectors (M-orthonormal) */
  const double* lambdas[3]; /* host, n[a] per-axis eigenvalues */
  const double* m_diag[3];  /* host, per-axis tridiagonal M_axis (may be NULL: no apply/residual) */
  const double* m_off[3];
  const double* a_diag[3];  /* host, per-axis tridiagonal A_axis */
  const double* a_off[3];
  int64_t time_chunk;       /* time slices per pipeline chunk for *_host calls (0 = auto) */
  /* Transform backend.  STKG_TRANSFORM_DENSE: X[a] is applied as a dense DMMA GEMM (any
   * EigPair).  STKG_TRANSFORM_P1_DST: the axes carry the closed-form uniform-P1 eigenbasis
   * X = S diag(mu^-1/2) of fem1d_matrices on a grid of spacing p1_h[a],
   * applied as an O(n log n) FP64 sine transform; needs n[a] + 1 a power of two in
   * [16, 2048]; X[a] is not read.  lambdas[a] are used by the recurrence in both modes. */
  int transform;
  double p1_h[3];
} stkg_heat_desc;

enum { STKG_TRANSFORM_DENSE = 0, STKG_TRANSFORM_P1_DST = 1 };

int stkg_heat_create(stkg_heat** plan, const stkg_heat_desc* desc, void* cuda_stream);
int stkg_heat_destroy(stkg_heat* plan);
/* Bytes of device workspace the plan holds (scratch + bases). */
int64_t stkg_heat_workspace_bytes(const stkg_heat* plan);
/* Which device schedule stkg_heat_solve runs for this plan (no reference counterpart; used by
 * bench.py and the tests to name the kernels they time):
 *   0  one transform pass per axis each way + the per-mode recurrence kernel
 *   1  time-marching fused axis-0 pass (forward DST, recurrence, inverse DST per slice)
 *   2  time-marching line-solve axis-0 pass (axis 0 is not transformed: one Toeplitz
 *      tridiagonal solve per column and slice; uniform time grids on uniform P1 axes) */
enum { STKG_SCHEDULE_SEPARATE = 0, STKG_SCHEDULE_FUSED_DST = 1, STKG_SCHEDULE_LINE_SOLVE = 2 };
int stkg_heat_schedule(const stkg_heat* plan);
/* solve_projected_heat_with (stk/sylvester.hpp:117-142): U = X Y~, Y~ from the per-mode
 * bidiagonal recurrence of X^T F.  F, U device, N_h x N_t column-major.  F is not
 * modified; U may not alias F.  STKG_SINGULARITY if |d_j + lambda_i c_j| < 1e-300. */
int stkg_heat_solve(stkg_heat* plan, const double* F, double* U);
/* Factored load F = L R^T (RHSFactors / LowRank, stk/rhs_sep.hpp:99-104,
 * stk/types.hpp:87-108): X^T F = (X^T L) R^T, so only the rank columns of L are transformed
 * and the recurrence forms each transformed column on the fly; F is never materialised.
 * L device n_x x rank, R device n_t x rank (column-major), 1 <= rank <= 16. */
int stkg_heat_solve_factored(stkg_heat* plan, int64_t rank, const double* L, const double* R,
                             double* U);
/* Same with HOST buffers (pinned or pageable): H2D of F, the solve and the D2H of U are
 * pipelined over time chunks (the recurrence is causal in time).  Synchronous. */
int stkg_heat_solve_host(stkg_heat* plan, const double* F_host, double* U_host);
/* KronOp::apply (stk/sylvester.hpp:32-38) of heat_kron_op: out = M U D + A U C. */
int stkg_heat_apply(stkg_heat* plan, const double* U, double* out);
/* ||F - KronOp::apply(U)||_F / ||F||_F with deterministic reductions (the residual of
 * stk/bench.hpp:508,524).  relres/fnorm are host outputs; synchronous. */
int stkg_heat_residual(stkg_heat* plan, const double* U, const double* F, double* relres,
                       double* fnorm);

/* Kernel-class timing for roofline evidence (no reference counterpart).  enable = 1 resets
 * and starts recording CUDA events around every launch on the plan's stream; enable = 0
 * stops, synchronizes and writes, per class [0] = basis transforms alone (DMMA GEMM or
 * sine-transform passes), [1] = kernels that run the modal recurrence (the scan, or the
 * fused axis-0 pass: transforms + recurrence), the summed device milliseconds (ms_out[2])
 * and launch counts (launches_out[2]).  Either output may be NULL.  While recording, 2D
 * solves run their passes back to back on the plan stream (no overlapped schedule), so the
 * per-launch times are those of the kernels alone. */
int stkg_heat_profile(stkg_heat* plan, int enable, double* ms_out, int64_t* launches_out);

/* ------------------------------------------------------------------ wave plans --- */
/* A wave plan holds WaveOperator (stk/outer_krylov.hpp:168-191) as banded factors and
 * TwoTermPrecond (stk/sylvester.hpp:153-181) as two EigPairs. */
typedef struct stkg_wave stkg_wave;

typedef struct stkg_wave_desc {
  int64_t nh;                 /* spatial dimension */
  int64_t nt;                 /* temporal dimension (number of temporal test functions) */
  const double* space_bands;  /* host, [M_h | A_h | Q_h], each 7*nh, layout as above */
  const double* time_bands;   /* host, [Q_t | D_t | M_t], each 7*nt */
  const double* Xs;           /* host, nh x nh: sym_gen_eig(Q_h, M_h).X (may be NULL) */
  const double* lambdas;      /* host, nh */
  const double* Xt;           /* host, nt x nt: sym_gen_eig(Q_t, M_t).X (may be NULL) */
  const double* thetas;       /* host, nt */
} stkg_wave_desc;

typedef struct stkg_gmres_config { /* GmresConfig (stk/outer_krylov.hpp:18-28) */
  double tol;                      /* default 1e-8 */
  int maxit;                       /* default 200 */
  int restart;                     /* 0 = full GMRES */
  int use_precond;                 /* 1 = right preconditioning by TwoTermPrecond */
} stkg_gmres_config;

typedef struct stkg_report {       /* SolveReport (stk/report.hpp:11-20) */
  int iterations;
  int mu_mem;
  int converged;
  int stagnated;
  double final_relres;
  double wall_time_s;
  double* rel_res_history;         /* host, caller-owned, capacity history_capacity (may be NULL) */
  int history_capacity;
  int history_length;
} stkg_report;

/* ------------------------------------------------------- rational Krylov (RKSM) --- */
typedef struct stkg_rksm_options { /* RksmOptions (stk/rksm.hpp:104-113) */
  double tol;                      /* default 1e-8 */
  int maxit;                       /* default 100 */
  int fixed_iters;                 /* > 0: preconditioner mode, exactly this many expansions */
  double trunc_tol;                /* default 1e-10 (truncation tolerance in that mode) */
} stkg_rksm_options;

/* rksm_solve (stk/rksm.hpp:127-234): rational Krylov Galerkin solve of the plan's heat
 * system M U D + A U C = F for a factored load F = L R^T (L device n_x x rank, R device
 * n_t x rank, column-major).  Shifted solves (A - sigma M)^-1 M are batched tridiagonal
 * solves in 1D and diagonal scalings between the plan's basis transforms in 2D/3D; block
 * orthogonalisation is tall-skinny GEMM passes; the spectral interval is the exact one of
 * the tensor pencil, widened by [1/2, 2] like estimate_spectral_interval (:21-51).  The
 * truncated solution is returned factored, U = U_left U_right^T (device n_x x cap and
 * n_t x cap), its rank in *rank_out.  Needs a plan created with the spatial factors. */
int stkg_heat_rksm(stkg_heat* plan, int64_t rank, const double* L, const double* R,
                   const stkg_rksm_options* opts, double* U_left, double* U_right, int64_t cap,
                   int64_t* rank_out, stkg_report* report);

/* ------------------------------------------------------- generic Krylov solvers --- */
/* Device-vector operator callback: the VecOp of stk/outer_krylov.hpp:30, i.e. the seam
 * run_wave_experiment passes lambdas through (stk/bench.hpp:667-673).  y = op(x) for
 * device vectors of length n, enqueued on cuda_stream; return STKG_OK or a status code
 * (a non-zero status aborts the solve and is returned by the solver). */
typedef int (*stkg_vec_op)(void* user, const double* x, double* y, void* cuda_stream);

/* gmres (stk/outer_krylov.hpp:75-164) over arbitrary device operators: right
 * preconditioning (precond may be NULL), full or restarted, Gram-Schmidt with one
 * re-orthogonalisation pass, Givens least squares, true final residual.  b, x device. */
int stkg_gmres_op(int64_t n, stkg_vec_op apply, void* apply_user, stkg_vec_op precond,
                  void* precond_user, const double* b, double* x, const stkg_gmres_config* cfg,
                  stkg_report* report, void* cuda_stream);
/* Preconditioned CG over device operators (both must be s.p.d.). */
int stkg_pcg_op(int64_t n, stkg_vec_op apply, void* apply_user, stkg_vec_op precond,
                void* precond_user, const double* b, double* x, double tol, int maxit,
                stkg_report* report, void* cuda_stream);

int stkg_wave_create(stkg_wave** plan, const stkg_wave_desc* desc, void* cuda_stream);
int stkg_wave_destroy(stkg_wave* plan);
/* WaveOperator::apply (stk/outer_krylov.hpp:178-186):
 * y = vec(M_h U Q_t^T + A_h U (D_t + D_t^T) + Q_h U M_t), x, y device, length nh*nt. */
int stkg_wave_apply(stkg_wave* plan, const double* x, double* y);
/* TwoTermPrecond::solve (stk/sylvester.hpp:168-176): W = X_s [(X_s^T V X_t) ./ (l_i + t_j)] X_t^T.
 * STKG_SOLVABILITY at create time if min(lambda) + min(theta) <= 0 (stk/sylvester.hpp:158-160). */
int stkg_two_term_solve(stkg_wave* plan, const double* v, double* w);
/* Space-modal, time-banded preconditioner (no reference counterpart; K2d):
 * P = M_h (x) Q_t + A' (x) E + Q_h (x) M_t with A_h replaced by its diagonal in the
 * TwoTermPrecond eigenbasis, A' = X_s^-T diag(x_i^T A_h x_i) X_s^-1.  Applied as
 * W = X_s [K_i^-1 rows of X_s^T V], K_i = Q_t + a_i (D_t + D_t^T) + lambda_i M_t (banded
 * Cholesky per spatial mode, factored at plan creation).  s.p.d.; STKG_DEFINITENESS at create
 * time if some K_i is not. */
int stkg_modal_banded_solve(stkg_wave* plan, const double* v, double* w);
/* The preconditioner stkg_gmres (use_precond = 1), stkg_pcg and stkg_wave_solve_refined
 * apply: 0 = TwoTermPrecond (default, the reference's), 1 = the modal banded one. */
int stkg_wave_set_precond(stkg_wave* plan, int kind);
/* gmres (stk/outer_krylov.hpp:75-164) with apply = WaveOperator, precond = TwoTermPrecond:
 * right-preconditioned Arnoldi, Gram-Schmidt with one re-orthogonalisation pass (run as
 * classical GS twice: tall-skinny GEMV passes), Givens least squares on the host.
 * b, x device.  x is overwritten (initial guess 0, as the reference). */
int stkg_gmres(stkg_wave* plan, const double* b, double* x, const stkg_gmres_config* cfg,
               stkg_report* report);
/* Preconditioned CG with the same preconditioner (no reference counterpart; valid
 * because the wave operator and TwoTermPrecond are both s.p.d.).
 * Stops on the recursively updated ||r||/||b|| <= tol; final_relres is the true one. */
int stkg_pcg(stkg_wave* plan, const double* b, double* x, double tol, int maxit,
             stkg_report* report);
/* r = b - B (x_hi + x_lo) evaluated in double-double arithmetic (error-free products of the
 * band coefficients, compensated sums), returned rounded to FP64 in r (device, may be NULL),
 * with ||r||_2 / ||b||_2 in *relres.  x_lo may be NULL (treated as 0).  SURVEY F5: at config
 * 4 the FP64-evaluated residual itself has an error floor near 1e-8..1e-7, so a 1e-10 bar
 * can only be checked (and met) with an extended-precision residual. */
int stkg_wave_residual_dd(stkg_wave* plan, const double* b, const double* x_hi,
                          const double* x_lo, double* r, double* relres);
/* Mixed-precision iterative refinement for the wave system: the solution
 * is kept as an unevaluated double-double sum x_hi + x_lo; each round computes the residual
 * in double-double (stkg_wave_residual_dd), solves B d = r with PCG to inner_tol, and adds d
 * with a two-sum.  Stops when the double-double relative residual is <= tol or after
 * max_refine corrections.  report: iterations = total PCG iterations; rel_res_history = the
 * double-double relative residual before each correction and at the end. */
int stkg_wave_solve_refined(stkg_wave* plan, const double* b, double* x_hi, double* x_lo,
                            double tol, int max_refine, double inner_tol, int inner_maxit,
                            stkg_report* report);

#ifdef __cplusplus
}
#endif

#endif /* STK_GPU_H */
