// Wave hot path: the very-weak space-time wave system
//     M_h U Q_t^T + A_h U (D_t + D_t^T) + Q_h U M_t = F        (stk/outer_krylov.hpp:178-186)
// solved by right-preconditioned full GMRES with the diagonalised two-term preconditioner
// M_h W Q_t^T + Q_h W M_t = V (stk/sylvester.hpp:153-181), plus a PCG performance path.
//   K5  banded Kronecker operator (7-diagonal spatial x 7-diagonal temporal factors)
//   K2  TwoTermPrecond::solve = 4 DMMA GEMMs with a fused divide-by-(lambda_i+theta_j)
//   K4  Arnoldi orthogonalisation as tall-skinny GEMV passes (classical GS, twice)
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "gemm_f64.cuh"
#include "krylov.cuh"

using namespace stkg;

namespace {
constexpr int kTerms = 3;
constexpr int kHalf = 3;  // half-bandwidth of the cubic-spline factors
constexpr int kBand = 2 * kHalf + 1;
}  // namespace

struct stkg_wave {
  int64_t nh = 0, nt = 0, N = 0;
  cudaStream_t stream = nullptr;
  // KronOp terms out = sum_p S_p U T_p^T (stk/sylvester.hpp:36): S = {M_h, A_h, Q_h},
  // T = {Q_t, E^T, M_t^T}, E = D_t + D_t^T (stk/outer_krylov.hpp:173).
  DevBuf S[kTerms], T[kTerms];
  bool has_precond = false;
  DevBuf Xs, XsT, lam, Xt, XtT, theta;
  DevBuf t1, t2;            // preconditioner temporaries (nh x nt)
  // space-modal, time-banded preconditioner (precond_kind 1, modal_banded_solve): per
  // spatial mode i the banded Cholesky factor of K_i = Q_t + a_i E + lambda_i M_t,
  // mb[k * N + i + nh j] = L_i(j, j - k) (k = 1..3), mb[i + nh j] = 1 / L_i(j, j)
  bool has_modal = false;
  int precond_kind = 0;      // 0 = TwoTermPrecond (the reference's), 1 = modal banded
  DevBuf mb;
  std::vector<double> modal_a;  // a_i = (X_s^T A_h X_s)_ii, host copy
  Krylov krylov;             // GMRES / PCG workspace (basis grows on demand)
  StreamKWork sk;            // stream-K GEMM workspace (1k^3 preconditioner products)
  DevBuf ref_r, ref_d;       // refinement residual / correction, kept across calls (a per-call
                             // cudaMalloc + cudaFree synchronises the device: 10 -> 64 ms
                             // swings for the config-4 refined solve)
  ~stkg_wave() {
    if (sk.partials) cudaFree(sk.partials);
    if (sk.flags) cudaFree(sk.flags);
  }
};

namespace {

// ------------------------------------------------------------------------------ K5 --
// Tile of TI (space) x TJ (time) outputs.  The U tile with a 3-wide halo on both axes and
// the band coefficients of the tile's rows/columns are staged in shared memory once; the
// temporal products V_p = U T_p^T are formed for the TI+6 halo rows, then the spatial
// bands are applied.  U and out each cross L2/HBM once (16 B/unknown).
constexpr int TI = 32, TJ = 16, KThreads = 256;
constexpr int TIH = TI + 2 * kHalf, TJH = TJ + 2 * kHalf;

__global__ void __launch_bounds__(KThreads) wave_apply_kernel(
    const double* __restrict__ U, double* __restrict__ out, int64_t nh, int64_t nt,
    const double* __restrict__ S0, const double* __restrict__ S1, const double* __restrict__ S2,
    const double* __restrict__ T0, const double* __restrict__ T1, const double* __restrict__ T2,
    const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double su[TJH][TIH];           // [time][space]
  __shared__ double sv[kTerms][TJ][TIH];    // temporal products
  __shared__ double st[kTerms][kBand][TJ];  // temporal band coefficients of the tile columns
  __shared__ double ss[kTerms][kBand][TI];  // spatial band coefficients of the tile rows
  const int64_t i0 = int64_t(blockIdx.x) * TI, j0 = int64_t(blockIdx.y) * TJ;
  for (int e = threadIdx.x; e < TJH * TIH; e += KThreads) {
    const int jj = e / TIH, ii = e % TIH;
    const int64_t gi = i0 + ii - kHalf, gj = j0 + jj - kHalf;
    su[jj][ii] = (gi >= 0 && gi < nh && gj >= 0 && gj < nt) ? U[gj * nh + gi] : 0.0;
  }
  for (int e = threadIdx.x; e < kTerms * kBand * TJ; e += KThreads) {
    const int t = e / (kBand * TJ), b = (e / TJ) % kBand, jj = e % TJ;
    const int64_t gj = j0 + jj;
    const double* T = t == 0 ? T0 : (t == 1 ? T1 : T2);
    st[t][b][jj] = gj < nt ? T[b * nt + gj] : 0.0;
  }
  for (int e = threadIdx.x; e < kTerms * kBand * TI; e += KThreads) {
    const int t = e / (kBand * TI), a = (e / TI) % kBand, ii = e % TI;
    const int64_t gi = i0 + ii;
    const double* S = t == 0 ? S0 : (t == 1 ? S1 : S2);
    ss[t][a][ii] = gi < nh ? S[a * nh + gi] : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < TJ * TIH; e += KThreads) {
    const int jj = e / TIH, ii = e % TIH;
    double u[kBand];
#pragma unroll
    for (int b = 0; b < kBand; ++b) u[b] = su[jj + b][ii];
#pragma unroll
    for (int t = 0; t < kTerms; ++t) {
      double acc = st[t][0][jj] * u[0];
#pragma unroll
      for (int b = 1; b < kBand; ++b) acc = fma(st[t][b][jj], u[b], acc);
      sv[t][jj][ii] = acc;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < TJ * TI; e += KThreads) {
    const int jj = e / TI, ii = e % TI;
    const int64_t gi = i0 + ii, gj = j0 + jj;
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < kTerms; ++t) {
      double part = ss[t][0][ii] * sv[t][jj][ii];
#pragma unroll
      for (int a = 1; a < kBand; ++a) part = fma(ss[t][a][ii], sv[t][jj][ii + a], part);
      acc = t == 0 ? part : acc + part;
    }
    if (gi < nh && gj < nt) out[gj * nh + gi] = acc;
  }
}

// ---------------------------------------------------- double-double residual (F5) --
// Error-free transformations written with the _rn intrinsics so that the compiler cannot
// contract them into FMAs.
struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, e};
}
__device__ __forceinline__ DD fast_two_sum(double a, double b) {  // |a| >= |b|
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  DD s = two_sum(a.hi, b.hi);
  const DD t = two_sum(a.lo, b.lo);
  s.lo = __dadd_rn(s.lo, t.hi);
  s = fast_two_sum(s.hi, s.lo);
  s.lo = __dadd_rn(s.lo, t.lo);
  return fast_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ DD dd_mul(DD a, DD b) {
  const double p = __dmul_rn(a.hi, b.hi);
  double e = fma(a.hi, b.hi, -p);                  // exact low part of a.hi * b.hi
  e = fma(a.hi, b.lo, e);
  e = fma(a.lo, b.hi, e);
  return fast_two_sum(p, e);
}

// r = b - sum_p S_p U T_p^T with U = xh + xl, out(i, j) = sum_p sum_a sum_b S_p[a][i]
// T_p[b][j] U(i + a - 3, j + b - 3) (the K5 stencil written per output), all in
// double-double.  One thread per output; called a few times per solve.
__global__ void __launch_bounds__(256) wave_residual_dd_kernel(
    const double* __restrict__ bvec, const double* __restrict__ xh, const double* __restrict__ xl,
    double* __restrict__ r, int64_t nh, int64_t nt, const double* __restrict__ S0,
    const double* __restrict__ S1, const double* __restrict__ S2, const double* __restrict__ T0,
    const double* __restrict__ T1, const double* __restrict__ T2) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= nh * nt) return;
  const int64_t i = e % nh, j = e / nh;
  const double* S[3] = {S0, S1, S2};
  const double* T[3] = {T0, T1, T2};
  DD acc = {0.0, 0.0};
  for (int p = 0; p < kTerms; ++p) {
    for (int bb = 0; bb < kBand; ++bb) {
      const int64_t jj = j + bb - kHalf;
      if (jj < 0 || jj >= nt) continue;
      const double tc = T[p][bb * nt + j];
      if (tc == 0.0) continue;
      for (int a = 0; a < kBand; ++a) {
        const int64_t ii = i + a - kHalf;
        if (ii < 0 || ii >= nh) continue;
        const double sc = S[p][a * nh + i];
        if (sc == 0.0) continue;
        const double cp = __dmul_rn(sc, tc);
        const DD coef = {cp, fma(sc, tc, -cp)};  // exact product of the two coefficients
        const int64_t o = jj * nh + ii;
        acc = dd_add(acc, dd_mul(coef, DD{xh[o], xl ? xl[o] : 0.0}));
      }
    }
  }
  const DD res = dd_add(DD{bvec[e], 0.0}, DD{-acc.hi, -acc.lo});
  r[e] = __dadd_rn(res.hi, res.lo);
}

// (xh, xl) += d as a double-double sum.
__global__ void dd_accumulate_kernel(double* __restrict__ xh, double* __restrict__ xl,
                                     const double* __restrict__ d, int64_t n) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const DD s = dd_add(DD{xh[e], xl[e]}, DD{d[e], 0.0});
    xh[e] = s.hi;
    xl[e] = s.lo;
  }
}

double residual_dd(stkg_wave& w, const double* b, const double* xh, const double* xl, double* r) {
  wave_residual_dd_kernel<<<static_cast<unsigned>(ceil_div(w.N, 256)), 256, 0, w.stream>>>(
      b, xh, xl, r, w.nh, w.nt, w.S[0].p, w.S[1].p, w.S[2].p, w.T[0].p, w.T[1].p, w.T[2].p);
  STKG_CUDA_CHECK(cudaGetLastError());
  const double nb = knorm(w.krylov, b);
  return nb > 0.0 ? knorm(w.krylov, r) / nb : 0.0;
}

std::vector<double> transpose(const double* X, int64_t n) {
  std::vector<double> t(static_cast<size_t>(n * n));
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) t[i * n + j] = X[j * n + i];
  return t;
}

// band of A^T from band of A: AT[d][j] = A[j + d - 3, j] = band_A[6 - d][j + d - 3]
std::vector<double> band_transpose(const double* band, int64_t n) {
  std::vector<double> out(static_cast<size_t>(kBand * n), 0.0);
  for (int d = 0; d < kBand; ++d)
    for (int64_t j = 0; j < n; ++j) {
      const int64_t i = j + d - kHalf;
      if (i >= 0 && i < n) out[d * n + j] = band[(kBand - 1 - d) * n + i];
    }
  return out;
}

// ------------------------------------------------------------------------ building blocks
void apply_op(stkg_wave& w, const double* x, double* y) {
  // (w.krylov.skip: device flag of a converged PCG; the kernel is a no-op once it is set)
  dim3 grid(static_cast<unsigned>(ceil_div(w.nh, TI)), static_cast<unsigned>(ceil_div(w.nt, TJ)));
  wave_apply_kernel<<<grid, KThreads, 0, w.stream>>>(x, y, w.nh, w.nt, w.S[0].p, w.S[1].p,
                                                    w.S[2].p, w.T[0].p, w.T[1].p, w.T[2].p,
                                                    w.krylov.skip);
  STKG_CUDA_CHECK(cudaGetLastError());
}

// ------------------------------------------------ space-modal time-banded preconditioner --
// P = M_h (x) Q_t + A' (x) E + Q_h (x) M_t with A_h replaced by A' = X_s^-T diag(a) X_s^-1,
// a_i = x_i^T A_h x_i (the diagonal of A_h in the TwoTermPrecond eigenbasis, which is
// X_s^T M_h X_s = I, X_s^T Q_h X_s = Lambda).  In that basis P is block diagonal: row i of
// W~ = X_s^-1 W solves the 7-banded s.p.d. time system K_i w~_i = (X_s^T V)_i with
// K_i = Q_t + a_i E + lambda_i M_t, so
//     P^-1 V = X_s [K_i^-1 rows of (X_s^T V)]    -- 2 GEMMs + n_h banded Cholesky solves
// (TwoTermPrecond drops the A_h (x) E term and needs 4 GEMMs).  A_h is nearly diagonal in
// that basis (off-diagonal mass 1-2% at n = 63..255, tools: DESIGN.md K2d), so P is almost
// B: PCG needs ~10 iterations at every size instead of TwoTermPrecond's ~1.3 sqrt-growth
// (537 at n = 255, 1370 at config 4).  P is s.p.d. whenever every K_i is (a_i > 0 since A_h
// is s.p.d.; the factorisation checks the pivots).
// One thread per spatial mode runs the forward and backward substitution over time; the
// loads of a block of U steps do not depend on the recurrence and are issued ahead.
template <int U>
struct BandBlock {  // one block of U steps of a mode's substitution: operands only
  double v[U], r[U], a[U], b[U], c[U];
};

__global__ void __launch_bounds__(32) modal_banded_solve_kernel(double* __restrict__ t,
                                                                const double* __restrict__ mb,
                                                                int64_t nh, int64_t nt,
                                                                const int* skip) {
  if (skip && *skip) return;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nh) return;
  const int64_t N = nh * nt;
  const double* rd = mb + i;
  const double* l1 = mb + N + i;
  const double* l2 = mb + 2 * N + i;
  const double* l3 = mb + 3 * N + i;
  double* col = t + i;
  constexpr int U = 8;
  const int64_t nb = nt / U;  // full blocks; the remainder runs unpipelined
  // forward: L y = v,  y_j = (v_j - L(j,j-1) y_{j-1} - L(j,j-2) y_{j-2} - L(j,j-3) y_{j-3}) / L(j,j)
  // The operands of block k+1 are loaded while block k's dependent chain runs (the chain
  // is two FP64 ops per step; unpipelined, every block waited a full L2 round trip).
  auto load_fwd = [&](int64_t k, BandBlock<U>& B) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t o = (k * U + u) * nh;
      B.v[u] = col[o];
      B.r[u] = __ldg(rd + o);
      B.a[u] = __ldg(l1 + o);
      B.b[u] = __ldg(l2 + o);
      B.c[u] = __ldg(l3 + o);
    }
  };
  double y1 = 0.0, y2 = 0.0, y3 = 0.0;
  {
    BandBlock<U> cur, nxt;
    if (nb > 0) load_fwd(0, cur);
    for (int64_t k = 0; k < nb; ++k) {
      if (k + 1 < nb) load_fwd(k + 1, nxt);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double y = (fma(-cur.c[u], y3, fma(-cur.b[u], y2, cur.v[u])) - cur.a[u] * y1) * cur.r[u];
        col[(k * U + u) * nh] = y;
        y3 = y2;
        y2 = y1;
        y1 = y;
      }
      cur = nxt;
    }
  }
  for (int64_t j = nb * U; j < nt; ++j) {
    const int64_t o = j * nh;
    const double y = (fma(-l3[o], y3, fma(-l2[o], y2, col[o])) - l1[o] * y1) * rd[o];
    col[o] = y;
    y3 = y2;
    y2 = y1;
    y1 = y;
  }
  // backward: L^T w = y,  w_j = (y_j - L(j+1,j) w_{j+1} - L(j+2,j) w_{j+2} - L(j+3,j) w_{j+3}) / L(j,j)
  double w1 = 0.0, w2 = 0.0, w3 = 0.0;
  const int64_t rem = nt - nb * U;  // the top rows (j >= nb U) first, unpipelined
  for (int64_t j = nt - 1; j >= nt - rem; --j) {
    const int64_t o = j * nh;
    const double a = j + 1 < nt ? l1[o + nh] : 0.0;
    const double b = j + 2 < nt ? l2[o + 2 * nh] : 0.0;
    const double c = j + 3 < nt ? l3[o + 3 * nh] : 0.0;
    const double w = (fma(-c, w3, fma(-b, w2, col[o])) - a * w1) * rd[o];
    col[o] = w;
    w3 = w2;
    w2 = w1;
    w1 = w;
  }
  auto load_bwd = [&](int64_t k, BandBlock<U>& B) {  // block k = rows k U + U - 1 .. k U
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = k * U + U - 1 - u, o = j * nh;
      B.v[u] = col[o];
      B.r[u] = __ldg(rd + o);
      B.a[u] = j + 1 < nt ? __ldg(l1 + o + nh) : 0.0;
      B.b[u] = j + 2 < nt ? __ldg(l2 + o + 2 * nh) : 0.0;
      B.c[u] = j + 3 < nt ? __ldg(l3 + o + 3 * nh) : 0.0;
    }
  };
  {
    BandBlock<U> cur, nxt;
    if (nb > 0) load_bwd(nb - 1, cur);
    for (int64_t k = nb - 1; k >= 0; --k) {
      if (k > 0) load_bwd(k - 1, nxt);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double w = (fma(-cur.c[u], w3, fma(-cur.b[u], w2, cur.v[u])) - cur.a[u] * w1) * cur.r[u];
        col[(k * U + U - 1 - u) * nh] = w;
        w3 = w2;
        w2 = w1;
        w1 = w;
      }
      cur = nxt;
    }
  }
}

// Parallel-in-time form of modal_banded_solve_kernel: a CTA of 32 x P threads takes 32
// consecutive modes (lane = mode, coalesced) and cuts each mode's time axis into P chunks
// (warp = chunk).  Each substitution is an order-3 linear recurrence on the state
// s_j = (y_j, y_{j-1}, y_{j-2}); per direction:
//   A  every chunk runs its rows from a zero state (giving e_c) and, in lockstep, the three
//      homogeneous runs from unit states (the columns of the chunk's 3 x 3 transfer G_c);
//   B  warp 0 chains the P chunks: s_in(c+1) = G_c s_in(c) + e_c;
//   C  every chunk reruns its rows from its true incoming state and stores them.
// The dependent chain per thread drops from 2 n_t steps to about 4 n_t / P, and the SM
// holds P times more warps.  Same arithmetic per step as the sequential kernel in pass C;
// the incoming states differ from the sequential ones only in rounding.
template <int P>
__global__ void __launch_bounds__(32 * P) modal_banded_solve_chunked_kernel(
    double* __restrict__ t, const double* __restrict__ mb, int64_t nh, int64_t nt,
    const int* skip) {
  if (skip && *skip) return;
  // per chunk and lane: e (3) and G columns (9); pass B overwrites e with the incoming state
  // (dynamic shared memory: P * 12 * 32 doubles, 96 KB at P = 32)
  extern __shared__ double sh_raw[];
  double (*sh)[12][32] = reinterpret_cast<double (*)[12][32]>(sh_raw);
  const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
  const int64_t i = int64_t(blockIdx.x) * 32 + lane;
  const bool act = i < nh;
  const int64_t N = nh * nt;
  const int64_t ii = act ? i : 0;
  const double* rd = mb + ii;
  const double* l1 = mb + N + ii;
  const double* l2 = mb + 2 * N + ii;
  const double* l3 = mb + 3 * N + ii;
  double* col = t + ii;
  const int64_t L = (nt + P - 1) / P, j0 = c * L, j1 = j0 + L < nt ? j0 + L : nt;

  // ---------------- forward: y_j = (v_j - l1 y_{j-1} - l2 y_{j-2} - l3 y_{j-3}) rd
  {
    double z[3] = {0, 0, 0}, g0[3] = {1, 0, 0}, g1[3] = {0, 1, 0}, g2[3] = {0, 0, 1};
    for (int64_t j = j0; j < j1; ++j) {
      const int64_t o = j * nh;
      const double a = act ? __ldg(l1 + o) : 0.0, b = act ? __ldg(l2 + o) : 0.0;
      const double cc = act ? __ldg(l3 + o) : 0.0, r = act ? __ldg(rd + o) : 0.0;
      const double v = act ? col[o] : 0.0;
      const double zn = (fma(-cc, z[2], fma(-b, z[1], v)) - a * z[0]) * r;
      const double h0 = -(fma(cc, g0[2], fma(b, g0[1], a * g0[0]))) * r;
      const double h1 = -(fma(cc, g1[2], fma(b, g1[1], a * g1[0]))) * r;
      const double h2 = -(fma(cc, g2[2], fma(b, g2[1], a * g2[0]))) * r;
      z[2] = z[1]; z[1] = z[0]; z[0] = zn;
      g0[2] = g0[1]; g0[1] = g0[0]; g0[0] = h0;
      g1[2] = g1[1]; g1[1] = g1[0]; g1[0] = h1;
      g2[2] = g2[1]; g2[1] = g2[0]; g2[0] = h2;
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      sh[c][q][lane] = z[q];
      sh[c][3 + q][lane] = g0[q];
      sh[c][6 + q][lane] = g1[q];
      sh[c][9 + q][lane] = g2[q];
    }
    __syncthreads();
    if (c == 0) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      for (int k = 0; k < P; ++k) {
        double ns[3];
#pragma unroll
        for (int q = 0; q < 3; ++q)
          ns[q] = sh[k][q][lane] + sh[k][3 + q][lane] * s0 + sh[k][6 + q][lane] * s1 +
                  sh[k][9 + q][lane] * s2;
        sh[k][0][lane] = s0;
        sh[k][1][lane] = s1;
        sh[k][2][lane] = s2;
        s0 = ns[0];
        s1 = ns[1];
        s2 = ns[2];
      }
    }
    __syncthreads();
    double y1 = sh[c][0][lane], y2 = sh[c][1][lane], y3 = sh[c][2][lane];
    if (act) {
      for (int64_t j = j0; j < j1; ++j) {
        const int64_t o = j * nh;
        const double y = (fma(-__ldg(l3 + o), y3, fma(-__ldg(l2 + o), y2, col[o])) -
                          __ldg(l1 + o) * y1) * __ldg(rd + o);
        col[o] = y;
        y3 = y2;
        y2 = y1;
        y1 = y;
      }
    }
    __syncthreads();  // every chunk's y is stored (the backward pass reads across chunks)
  }
  // ---------------- backward: w_j = (y_j - L(j+1,j) w_{j+1} - L(j+2,j) w_{j+2} - L(j+3,j) w_{j+3}) rd
  {
    auto coef = [&](int64_t j, double& a, double& b, double& cc, double& r) {
      const int64_t o = j * nh;
      a = (act && j + 1 < nt) ? __ldg(l1 + o + nh) : 0.0;
      b = (act && j + 2 < nt) ? __ldg(l2 + o + 2 * nh) : 0.0;
      cc = (act && j + 3 < nt) ? __ldg(l3 + o + 3 * nh) : 0.0;
      r = act ? __ldg(rd + o) : 0.0;
    };
    double z[3] = {0, 0, 0}, g0[3] = {1, 0, 0}, g1[3] = {0, 1, 0}, g2[3] = {0, 0, 1};
    for (int64_t j = j1 - 1; j >= j0; --j) {
      double a, b, cc, r;
      coef(j, a, b, cc, r);
      const double v = act ? col[j * nh] : 0.0;
      const double zn = (fma(-cc, z[2], fma(-b, z[1], v)) - a * z[0]) * r;
      const double h0 = -(fma(cc, g0[2], fma(b, g0[1], a * g0[0]))) * r;
      const double h1 = -(fma(cc, g1[2], fma(b, g1[1], a * g1[0]))) * r;
      const double h2 = -(fma(cc, g2[2], fma(b, g2[1], a * g2[0]))) * r;
      z[2] = z[1]; z[1] = z[0]; z[0] = zn;
      g0[2] = g0[1]; g0[1] = g0[0]; g0[0] = h0;
      g1[2] = g1[1]; g1[1] = g1[0]; g1[0] = h1;
      g2[2] = g2[1]; g2[1] = g2[0]; g2[0] = h2;
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      sh[c][q][lane] = z[q];
      sh[c][3 + q][lane] = g0[q];
      sh[c][6 + q][lane] = g1[q];
      sh[c][9 + q][lane] = g2[q];
    }
    __syncthreads();
    if (c == 0) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      for (int k = P - 1; k >= 0; --k) {
        double ns[3];
#pragma unroll
        for (int q = 0; q < 3; ++q)
          ns[q] = sh[k][q][lane] + sh[k][3 + q][lane] * s0 + sh[k][6 + q][lane] * s1 +
                  sh[k][9 + q][lane] * s2;
        sh[k][0][lane] = s0;
        sh[k][1][lane] = s1;
        sh[k][2][lane] = s2;
        s0 = ns[0];
        s1 = ns[1];
        s2 = ns[2];
      }
    }
    __syncthreads();
    double w1 = sh[c][0][lane], w2 = sh[c][1][lane], w3 = sh[c][2][lane];
    if (act) {
      for (int64_t j = j1 - 1; j >= j0; --j) {
        double a, b, cc, r;
        coef(j, a, b, cc, r);
        const int64_t o = j * nh;
        const double w = (fma(-cc, w3, fma(-b, w2, col[o])) - a * w1) * r;
        col[o] = w;
        w3 = w2;
        w2 = w1;
        w1 = w;
      }
    }
  }
}

// Host setup of the modal banded preconditioner: a_i, the banded Cholesky factors of every
// K_i (symmetrised: the spline Gram bands are symmetric only to rounding).
void build_modal_banded(stkg_wave& w, const double* space_bands, const double* time_bands,
                        const double* Xs, const double* lambdas) {
  const int64_t nh = w.nh, nt = w.nt, N = w.N;
  const double* Ab = space_bands + kBand * nh;  // A_h band
  w.modal_a.assign(static_cast<size_t>(nh), 0.0);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < nh; ++i) {
    const double* x = Xs + i * nh;
    double acc = 0.0;
    for (int64_t r = 0; r < nh; ++r) {
      double ax = 0.0;
      for (int d = 0; d < kBand; ++d) {
        const int64_t c = r + d - kHalf;
        if (c >= 0 && c < nh) ax += Ab[d * nh + r] * x[c];
      }
      acc += x[r] * ax;
    }
    w.modal_a[i] = acc;
  }
  const double* Qb = time_bands;
  const double* Db = time_bands + kBand * nt;
  const double* Mb = time_bands + 2 * kBand * nt;
  auto band = [&](const double* b, int64_t j, int off) {  // matrix entry (j, j + off)
    const int64_t c = j + off;
    return (c >= 0 && c < nt) ? b[(off + kHalf) * nt + j] : 0.0;
  };
  std::vector<double> host(static_cast<size_t>(4 * N), 0.0);
  int bad = 0;
  double bad_a = 0.0;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < nh; ++i) {
    const double a = w.modal_a[i], lam = lambdas[i];
    // K(j, j - k) for k = 0..3, symmetrised
    auto K = [&](int64_t j, int k) {
      const int64_t c = j - k;
      if (c < 0) return 0.0;
      const double e1 = band(Db, j, -k) + band(Db, c, k);  // E(j,c) = D(j,c) + D(c,j)
      const double e2 = band(Db, c, k) + band(Db, j, -k);  // E(c,j)
      const double kjc = band(Qb, j, -k) + a * e1 + lam * band(Mb, j, -k);
      const double kcj = band(Qb, c, k) + a * e2 + lam * band(Mb, c, k);
      return 0.5 * (kjc + kcj);
    };
    std::vector<double> L(static_cast<size_t>(4 * nt), 0.0);  // L[k * nt + j] = L(j, j - k)
    bool ok = true;
    for (int64_t j = 0; j < nt && ok; ++j) {
      for (int k = 3; k >= 1; --k) {  // L(j, c), c = j - k, in increasing c
        const int64_t c = j - k;
        if (c < 0) continue;
        double sum = K(j, k);
        for (int m = k + 1; m <= 3; ++m)  // columns c' = j - m < c shared by rows j and c
          if (j - m >= 0 && (m - k) <= 3) sum -= L[m * nt + j] * L[(m - k) * nt + c];
        L[k * nt + j] = sum / L[c];  // L(c, c) stored at L[0 * nt + c]
      }
      double d = K(j, 0);
      for (int k = 1; k <= 3; ++k) d -= L[k * nt + j] * L[k * nt + j];
      if (!(d > 0.0)) {
        ok = false;
        break;
      }
      L[j] = std::sqrt(d);
    }
    if (!ok) {
#pragma omp critical
      {
        bad = 1;
        bad_a = a;
      }
      continue;
    }
    for (int64_t j = 0; j < nt; ++j) {
      host[static_cast<size_t>(i + nh * j)] = 1.0 / L[j];
      for (int k = 1; k <= 3; ++k) host[static_cast<size_t>(k * N + i + nh * j)] = L[k * nt + j];
    }
  }
  if (bad) {
    char buf[160];
    snprintf(buf, sizeof buf, "modal banded preconditioner: K_i not s.p.d. (a_i = %g)", bad_a);
    throw Error(STKG_DEFINITENESS, buf);
  }
  w.mb.alloc(4 * N);
  w.mb.upload(host.data(), 4 * N, w.stream);
  STKG_CUDA_CHECK(cudaStreamSynchronize(w.stream));
  w.has_modal = true;
}

void modal_banded_solve(stkg_wave& w, const double* v, double* out) {
  const int64_t nh = w.nh, nt = w.nt;
  GemmProblem p;
  p.skip = w.krylov.skip;
  // t1 = Xs^T V
  p.M = nh; p.K = nh; p.N = nt;
  p.A = w.XsT.p; p.lda = nh; p.B = v; p.ldb = nh; p.C = w.t1.p; p.ldc = nh;
  launch_gemm_streamk(p, EpiStore{}, w.stream, w.sk);
  // rows of t1 <- K_i^-1 rows (STKG_MB_CHUNKS: time chunks per mode, 1 = sequential kernel)
  static const int chunks = [] {
    const char* e = std::getenv("STKG_MB_CHUNKS");
    return e ? std::atoi(e) : 32;
  }();
  const unsigned g32 = static_cast<unsigned>(ceil_div(nh, 32));
  auto chunked = [&](auto pc) {
    constexpr int P = decltype(pc)::value;
    constexpr int smem = P * 12 * 32 * int(sizeof(double));
    static const bool configured = [] {
      STKG_CUDA_CHECK(cudaFuncSetAttribute(modal_banded_solve_chunked_kernel<P>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      return true;
    }();
    (void)configured;
    modal_banded_solve_chunked_kernel<P><<<g32, 32 * P, smem, w.stream>>>(w.t1.p, w.mb.p, nh, nt,
                                                                          w.krylov.skip);
  };
  if (chunks >= 32 && nt >= 32 * 16)
    chunked(std::integral_constant<int, 32>{});
  else if (chunks >= 16 && nt >= 16 * 16)
    chunked(std::integral_constant<int, 16>{});
  else if (chunks >= 8 && nt >= 8 * 16)
    chunked(std::integral_constant<int, 8>{});
  else
    modal_banded_solve_kernel<<<g32, 32, 0, w.stream>>>(w.t1.p, w.mb.p, nh, nt, w.krylov.skip);
  STKG_CUDA_CHECK(cudaGetLastError());
  // out = Xs t1
  p.M = nh; p.K = nh; p.N = nt;
  p.A = w.Xs.p; p.lda = nh; p.B = w.t1.p; p.ldb = nh; p.C = out; p.ldc = nh;
  launch_gemm_streamk(p, EpiStore{}, w.stream, w.sk);
}

void two_term_solve(stkg_wave& w, const double* v, double* out) {
  const int64_t nh = w.nh, nt = w.nt;
  GemmProblem p;
  p.skip = w.krylov.skip;
  // t1 = Xs^T V   (stk/sylvester.hpp:171, evaluated left to right as Eigen does)
  p.M = nh; p.K = nh; p.N = nt;
  p.A = w.XsT.p; p.lda = nh; p.B = v; p.ldb = nh; p.C = w.t1.p; p.ldc = nh;
  launch_gemm_streamk(p, EpiStore{}, w.stream, w.sk);
  // t2 = (t1 Xt) ./ (lambda_i + theta_j)   (:172-174)
  p.M = nh; p.K = nt; p.N = nt;
  p.A = w.t1.p; p.lda = nh; p.B = w.Xt.p; p.ldb = nt; p.C = w.t2.p; p.ldc = nh;
  launch_gemm_streamk(p, EpiDivide{w.lam.p, w.theta.p}, w.stream, w.sk);
  // t1 = Xs t2 ; out = t1 Xt^T   (:175)
  p.M = nh; p.K = nh; p.N = nt;
  p.A = w.Xs.p; p.lda = nh; p.B = w.t2.p; p.ldb = nh; p.C = w.t1.p; p.ldc = nh;
  launch_gemm_streamk(p, EpiStore{}, w.stream, w.sk);
  p.M = nh; p.K = nt; p.N = nt;
  p.A = w.t1.p; p.lda = nh; p.B = w.XtT.p; p.ldb = nt; p.C = out; p.ldc = nh;
  launch_gemm_streamk(p, EpiStore{}, w.stream, w.sk);
}

// The plan's preconditioner for GMRES / PCG / refinement.
void precond_solve(stkg_wave& w, const double* v, double* out) {
  if (w.precond_kind == 1) return modal_banded_solve(w, v, out);
  two_term_solve(w, v, out);
}

}  // namespace

extern "C" {

int stkg_wave_create(stkg_wave** out, const stkg_wave_desc* desc, void* cuda_stream) {
  return guarded([&] {
    STKG_REQUIRE(out && desc, STKG_ARGUMENT, "stkg_wave_create: null argument");
    *out = nullptr;
    STKG_REQUIRE(desc->nh >= 1 && desc->nt >= 1, STKG_ARGUMENT, "stkg_wave_create: bad sizes");
    STKG_REQUIRE(desc->space_bands && desc->time_bands, STKG_ARGUMENT,
                 "stkg_wave_create: missing bands");
    auto w = std::make_unique<stkg_wave>();
    w->nh = desc->nh;
    w->nt = desc->nt;
    w->N = w->nh * w->nt;
    w->stream = static_cast<cudaStream_t>(cuda_stream);
    cudaStream_t s = w->stream;
    const int64_t nh = w->nh, nt = w->nt;
    const double* sb = desc->space_bands;
    const double* tb = desc->time_bands;  // [Q_t | D_t | M_t]
    for (int t = 0; t < kTerms; ++t) {
      w->S[t].alloc(kBand * nh);
      w->S[t].upload(sb + t * kBand * nh, kBand * nh, s);
    }
    // T_0 = Q_t (term M_h U Q_t^T); T_1 = E^T with E = D + D^T; T_2 = M_t^T (U M_t = U (M_t^T)^T)
    std::vector<double> e(static_cast<size_t>(kBand * nt), 0.0);
    {
      const double* d = tb + kBand * nt;
      const auto dT = band_transpose(d, nt);
      for (size_t k = 0; k < e.size(); ++k) e[k] = d[k] + dT[k];  // D(i,j) + D(j,i)
    }
    const auto eT = band_transpose(e.data(), nt);
    const auto mT = band_transpose(tb + 2 * kBand * nt, nt);
    const double* th[kTerms] = {tb, eT.data(), mT.data()};
    for (int t = 0; t < kTerms; ++t) {
      w->T[t].alloc(kBand * nt);
      w->T[t].upload(th[t], kBand * nt, s);
    }
    if (desc->Xs && desc->Xt && desc->lambdas && desc->thetas) {
      double lmin = desc->lambdas[0], tmin = desc->thetas[0];
      for (int64_t i = 0; i < nh; ++i) lmin = std::min(lmin, desc->lambdas[i]);
      for (int64_t j = 0; j < nt; ++j) tmin = std::min(tmin, desc->thetas[j]);
      STKG_REQUIRE(lmin + tmin > 0.0, STKG_SOLVABILITY,
                   "TwoTermPrecond: lambda_i + theta_j <= 0, system not solvable");
      w->has_precond = true;
      const auto xsT = transpose(desc->Xs, nh);
      const auto xtT = transpose(desc->Xt, nt);
      w->Xs.alloc(nh * nh);
      w->Xs.upload(desc->Xs, nh * nh, s);
      w->XsT.alloc(nh * nh);
      w->XsT.upload(xsT.data(), nh * nh, s);
      w->Xt.alloc(nt * nt);
      w->Xt.upload(desc->Xt, nt * nt, s);
      w->XtT.alloc(nt * nt);
      w->XtT.upload(xtT.data(), nt * nt, s);
      w->lam.alloc(nh);
      w->lam.upload(desc->lambdas, nh, s);
      w->theta.alloc(nt);
      w->theta.upload(desc->thetas, nt, s);
      w->t1.alloc(w->N);
      w->t2.alloc(w->N);
      build_modal_banded(*w, sb, tb, desc->Xs, desc->lambdas);
    }
    STKG_CUDA_CHECK(cudaStreamSynchronize(s));  // host temporaries die here
    w->krylov.N = w->N;
    w->krylov.stream = s;
    *out = w.release();
  });
}

int stkg_wave_destroy(stkg_wave* w) {
  return guarded([&] {
    if (!w) return;
    if (w->stream) cudaStreamSynchronize(w->stream);
    else cudaDeviceSynchronize();
    delete w;
  });
}

int stkg_wave_apply(stkg_wave* w, const double* x, double* y) {
  return guarded([&] {
    STKG_REQUIRE(w && x && y, STKG_ARGUMENT, "WaveOperator: null argument");
    STKG_REQUIRE(x != y, STKG_ARGUMENT, "WaveOperator: y may not alias x");
    apply_op(*w, x, y);
  });
}

int stkg_two_term_solve(stkg_wave* w, const double* v, double* out) {
  return guarded([&] {
    STKG_REQUIRE(w && v && out, STKG_ARGUMENT, "TwoTermPrecond::solve: null argument");
    STKG_REQUIRE(w->has_precond, STKG_ARGUMENT,
                 "TwoTermPrecond::solve: plan was created without eigenpairs");
    two_term_solve(*w, v, out);
  });
}

int stkg_wave_set_precond(stkg_wave* w, int kind) {
  return guarded([&] {
    STKG_REQUIRE(w, STKG_ARGUMENT, "set_precond: null plan");
    STKG_REQUIRE(kind == 0 || kind == 1, STKG_ARGUMENT, "set_precond: kind must be 0 or 1");
    STKG_REQUIRE(w->has_precond && (kind == 0 || w->has_modal), STKG_ARGUMENT,
                 "set_precond: plan was created without eigenpairs");
    w->precond_kind = kind;
  });
}

int stkg_modal_banded_solve(stkg_wave* w, const double* v, double* out) {
  return guarded([&] {
    STKG_REQUIRE(w && v && out, STKG_ARGUMENT, "modal_banded_solve: null argument");
    STKG_REQUIRE(w->has_modal, STKG_ARGUMENT,
                 "modal_banded_solve: plan was created without eigenpairs");
    modal_banded_solve(*w, v, out);
  });
}

// gmres (stk/outer_krylov.hpp:75-164) with apply = WaveOperator and precond =
// TwoTermPrecond, the pairing run_wave_experiment passes (stk/bench.hpp:667-673).
int stkg_gmres(stkg_wave* wv, const double* b, double* x, const stkg_gmres_config* cfg_in,
               stkg_report* rep) {
  return guarded([&] {
    STKG_REQUIRE(wv && b && x, STKG_ARGUMENT, "gmres: null argument");
    const stkg_gmres_config cfg = cfg_in ? *cfg_in : stkg_gmres_config{1e-8, 200, 0, 1};
    const bool use_p = cfg.use_precond != 0;
    STKG_REQUIRE(!use_p || wv->has_precond, STKG_ARGUMENT, "gmres: no preconditioner in plan");
    stkg_wave& w = *wv;
    const DevOp apply = [&](const double* in, double* out) { apply_op(w, in, out); };
    const DevOp precond = [&](const double* in, double* out) { precond_solve(w, in, out); };
    gmres_run(w.krylov, apply, use_p ? &precond : nullptr, b, x, cfg, rep);
  });
}

// Preconditioned CG with TwoTermPrecond (B and P s.p.d.).
int stkg_pcg(stkg_wave* wv, const double* b, double* x, double tol, int maxit,
             stkg_report* rep) {
  return guarded([&] {
    STKG_REQUIRE(wv && b && x, STKG_ARGUMENT, "pcg: null argument");
    STKG_REQUIRE(wv->has_precond, STKG_ARGUMENT, "pcg: no preconditioner in plan");
    stkg_wave& w = *wv;
    const DevOp apply = [&](const double* in, double* out) { apply_op(w, in, out); };
    const DevOp precond = [&](const double* in, double* out) { precond_solve(w, in, out); };
    pcg_run(w.krylov, apply, precond, b, x, tol, maxit, rep);
  });
}

int stkg_wave_residual_dd(stkg_wave* wv, const double* b, const double* x_hi,
                          const double* x_lo, double* r, double* relres) {
  return guarded([&] {
    STKG_REQUIRE(wv && b && x_hi && relres, STKG_ARGUMENT, "residual_dd: null argument");
    stkg_wave& w = *wv;
    w.krylov.ensure(0, 0);
    double* rr = r;
    if (!rr) {
      if (w.ref_r.n < static_cast<size_t>(w.N)) w.ref_r.alloc(w.N);
      rr = w.ref_r.p;
    }
    *relres = residual_dd(w, b, x_hi, x_lo, rr);
  });
}

int stkg_wave_solve_refined(stkg_wave* wv, const double* b, double* x_hi, double* x_lo,
                            double tol, int max_refine, double inner_tol, int inner_maxit,
                            stkg_report* rep) {
  return guarded([&] {
    STKG_REQUIRE(wv && b && x_hi && x_lo, STKG_ARGUMENT, "solve_refined: null argument");
    STKG_REQUIRE(wv->has_precond, STKG_ARGUMENT, "solve_refined: no preconditioner in plan");
    STKG_REQUIRE(max_refine >= 0 && inner_maxit >= 1, STKG_ARGUMENT,
                 "solve_refined: bad iteration limits");
    const auto t0 = std::chrono::steady_clock::now();
    stkg_wave& w = *wv;
    w.krylov.ensure(0, 0);
    const DevOp apply = [&](const double* in, double* out) { apply_op(w, in, out); };
    const DevOp precond = [&](const double* in, double* out) { precond_solve(w, in, out); };
    if (w.ref_r.n < static_cast<size_t>(w.N)) w.ref_r.alloc(w.N);
    if (w.ref_d.n < static_cast<size_t>(w.N)) w.ref_d.alloc(w.N);
    DevBuf& r = w.ref_r;
    DevBuf& d = w.ref_d;
    STKG_CUDA_CHECK(cudaMemsetAsync(x_hi, 0, sizeof(double) * w.N, w.stream));
    STKG_CUDA_CHECK(cudaMemsetAsync(x_lo, 0, sizeof(double) * w.N, w.stream));
    int total = 0, len = 0;
    double relres = 1.0;
    bool converged = false;
    auto push = [&](double v) {
      if (rep && rep->rel_res_history && len < rep->history_capacity) rep->rel_res_history[len] = v;
      ++len;
    };
    for (int k = 0;; ++k) {
      relres = residual_dd(w, b, x_hi, x_lo, r.p);
      push(relres);
      if (relres <= tol) {
        converged = true;
        break;
      }
      if (k == max_refine) break;
      stkg_report inner{};
      pcg_run(w.krylov, apply, precond, r.p, d.p, inner_tol, inner_maxit, &inner);
      total += inner.iterations;
      dd_accumulate_kernel<<<num_sms() * 8, 256, 0, w.stream>>>(x_hi, x_lo, d.p, w.N);
      STKG_CUDA_CHECK(cudaGetLastError());
    }
    STKG_CUDA_CHECK(cudaStreamSynchronize(w.stream));
    if (rep) {
      rep->iterations = total;
      rep->converged = converged ? 1 : 0;
      rep->stagnated = 0;
      rep->final_relres = relres;
      rep->history_length = len;
      rep->mu_mem = 0;
      rep->wall_time_s =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

}  // extern "C"
