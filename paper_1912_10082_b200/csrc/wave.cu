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
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "gemm_f64.cuh"

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
  DevBuf partials, scalars;
  double* pinned = nullptr;  // host mirror of reduction results
  int pinned_cap = 0;
  // Krylov workspace
  DevBuf V;                  // basis, N x cap (column-major)
  int64_t v_cap = 0;
  DevBuf w, z, r, p, q, xk;  // work vectors
  DevBuf hvec;               // device copy of Gram-Schmidt coefficients
};

namespace {

// ------------------------------------------------------------------------------ K5 --
// Tile of TI (space) x TJ (time) outputs; U tile with a 3-wide halo on both axes is staged
// in shared memory once; the temporal products V_p = U T_p^T are formed for the TI+6 halo
// rows, then the spatial bands are applied.  U and out each cross HBM/L2 once.
constexpr int TI = 64, TJ = 16, KThreads = 256;

__global__ void __launch_bounds__(KThreads) wave_apply_kernel(
    const double* __restrict__ U, double* __restrict__ out, int64_t nh, int64_t nt,
    const double* __restrict__ S0, const double* __restrict__ S1, const double* __restrict__ S2,
    const double* __restrict__ T0, const double* __restrict__ T1, const double* __restrict__ T2) {
  __shared__ double su[TJ + 2 * kHalf][TI + 2 * kHalf];  // [time][space]
  __shared__ double sv[kTerms][TJ][TI + 2 * kHalf];
  const int64_t i0 = int64_t(blockIdx.x) * TI, j0 = int64_t(blockIdx.y) * TJ;
  for (int e = threadIdx.x; e < (TJ + 2 * kHalf) * (TI + 2 * kHalf); e += KThreads) {
    const int jj = e / (TI + 2 * kHalf), ii = e % (TI + 2 * kHalf);
    const int64_t gi = i0 + ii - kHalf, gj = j0 + jj - kHalf;
    su[jj][ii] = (gi >= 0 && gi < nh && gj >= 0 && gj < nt) ? U[gj * nh + gi] : 0.0;
  }
  __syncthreads();
  const double* Tp[kTerms] = {T0, T1, T2};
  for (int e = threadIdx.x; e < TJ * (TI + 2 * kHalf); e += KThreads) {
    const int jj = e / (TI + 2 * kHalf), ii = e % (TI + 2 * kHalf);
    const int64_t gj = j0 + jj;
#pragma unroll
    for (int t = 0; t < kTerms; ++t) {
      double acc = 0.0;
      if (gj < nt) {
#pragma unroll
        for (int b = 0; b < kBand; ++b) acc += su[jj + b][ii] * __ldg(Tp[t] + b * nt + gj);
      }
      sv[t][jj][ii] = acc;
    }
  }
  __syncthreads();
  const double* Sp[kTerms] = {S0, S1, S2};
  for (int e = threadIdx.x; e < TJ * TI; e += KThreads) {
    const int jj = e / TI, ii = e % TI;
    const int64_t gi = i0 + ii, gj = j0 + jj;
    if (gi >= nh || gj >= nt) continue;
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < kTerms; ++t)
#pragma unroll
      for (int a = 0; a < kBand; ++a) acc += __ldg(Sp[t] + a * nh + gi) * sv[t][jj][ii + a];
    out[gj * nh + gi] = acc;
  }
}

// ---------------------------------------------------------------------- vector ops --
// Deterministic dot products: fixed grid, fixed per-thread order, block tree, then one
// block sums the partials in index order.
__global__ void __launch_bounds__(kReduceThreads) dot_partials_kernel(
    const double* __restrict__ x, const double* __restrict__ y, int64_t n,
    double* __restrict__ partials) {
  __shared__ double red[kReduceThreads / 32];
  double s = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kReduceThreads + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * kReduceThreads)
    s += x[i] * y[i];
  s = block_sum<kReduceThreads>(s, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kReduceThreads) sum_partials_kernel(
    const double* __restrict__ partials, int count, int ncols, double* __restrict__ out) {
  // column c of a count x ncols partials matrix (partials[c * count + b])
  __shared__ double red[kReduceThreads / 32];
  const int c = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < count; b += kReduceThreads) s += partials[int64_t(c) * count + b];
  s = block_sum<kReduceThreads>(s, red);
  if (threadIdx.x == 0) out[c] = s;
}

// h_c = V(:,c)^T w for c in [0, m): blockIdx.y picks a group of 4 columns, blockIdx.x a
// fixed row slice; partials[c * gridDim.x + blockIdx.x].
constexpr int kGemvCols = 4;
__global__ void __launch_bounds__(kReduceThreads) gemv_t_kernel(
    const double* __restrict__ V, int64_t N, int m, const double* __restrict__ w,
    double* __restrict__ partials) {
  __shared__ double red[kReduceThreads / 32];
  const int c0 = blockIdx.y * kGemvCols;
  double s[kGemvCols] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = int64_t(blockIdx.x) * kReduceThreads + threadIdx.x; i < N;
       i += int64_t(gridDim.x) * kReduceThreads) {
    const double wi = w[i];
#pragma unroll
    for (int c = 0; c < kGemvCols; ++c)
      if (c0 + c < m) s[c] += V[int64_t(c0 + c) * N + i] * wi;
  }
#pragma unroll
  for (int c = 0; c < kGemvCols; ++c) {
    const double t = block_sum<kReduceThreads>(s[c], red);
    if (threadIdx.x == 0 && c0 + c < m) partials[int64_t(c0 + c) * gridDim.x + blockIdx.x] = t;
  }
}

// w -= V h (h on the device, m columns); also accumulates ||w||^2 partials when asked.
__global__ void __launch_bounds__(kReduceThreads) gemv_n_update_kernel(
    const double* __restrict__ V, int64_t N, int m, const double* __restrict__ h,
    double* __restrict__ w, double* __restrict__ partials) {
  __shared__ double red[kReduceThreads / 32];
  double nrm = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kReduceThreads + threadIdx.x; i < N;
       i += int64_t(gridDim.x) * kReduceThreads) {
    double acc = w[i];
    int c = 0;
    for (; c + 4 <= m; c += 4) {
      const double v0 = V[int64_t(c) * N + i], v1 = V[int64_t(c + 1) * N + i];
      const double v2 = V[int64_t(c + 2) * N + i], v3 = V[int64_t(c + 3) * N + i];
      acc -= h[c] * v0;
      acc -= h[c + 1] * v1;
      acc -= h[c + 2] * v2;
      acc -= h[c + 3] * v3;
    }
    for (; c < m; ++c) acc -= h[c] * V[int64_t(c) * N + i];
    w[i] = acc;
    nrm += acc * acc;
  }
  if (partials) {
    nrm = block_sum<kReduceThreads>(nrm, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = nrm;
  }
}

__global__ void scale_copy_kernel(const double* __restrict__ x, double a, double* __restrict__ y,
                                  int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    y[i] = a * x[i];
}

// y = x - y  (residual r = b - Ax with Ax in y)
__global__ void sub_from_kernel(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    y[i] = x[i] - y[i];
}

// y += x
__global__ void add_kernel(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    y[i] += x[i];
}

// PCG update: x += a p; r -= a q; partial ||r||^2
__global__ void __launch_bounds__(kReduceThreads) cg_update_kernel(
    double a, const double* __restrict__ p, const double* __restrict__ q, double* __restrict__ x,
    double* __restrict__ r, int64_t n, double* __restrict__ partials) {
  __shared__ double red[kReduceThreads / 32];
  double s = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kReduceThreads + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * kReduceThreads) {
    x[i] += a * p[i];
    const double ri = r[i] - a * q[i];
    r[i] = ri;
    s += ri * ri;
  }
  s = block_sum<kReduceThreads>(s, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// p = z + b p
__global__ void xpby_kernel(const double* __restrict__ z, double b, double* __restrict__ p,
                            int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = z[i] + b * p[i];
}

constexpr unsigned kEwBlocks = 148 * 8;

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

void ensure_pinned(stkg_wave& w, int count) {
  if (count <= w.pinned_cap) return;
  if (w.pinned) cudaFreeHost(w.pinned);
  w.pinned = nullptr;
  STKG_CUDA_CHECK(cudaMallocHost(&w.pinned, sizeof(double) * count));
  w.pinned_cap = count;
}

// ------------------------------------------------------------------------ building blocks
void apply_op(stkg_wave& w, const double* x, double* y) {
  dim3 grid(static_cast<unsigned>(ceil_div(w.nh, TI)), static_cast<unsigned>(ceil_div(w.nt, TJ)));
  wave_apply_kernel<<<grid, KThreads, 0, w.stream>>>(x, y, w.nh, w.nt, w.S[0].p, w.S[1].p,
                                                    w.S[2].p, w.T[0].p, w.T[1].p, w.T[2].p);
  STKG_CUDA_CHECK(cudaGetLastError());
}

void precond_solve(stkg_wave& w, const double* v, double* out) {
  const int64_t nh = w.nh, nt = w.nt;
  GemmProblem p;
  // t1 = Xs^T V   (stk/sylvester.hpp:171, evaluated left to right as Eigen does)
  p.M = nh; p.K = nh; p.N = nt;
  p.A = w.XsT.p; p.lda = nh; p.B = v; p.ldb = nh; p.C = w.t1.p; p.ldc = nh;
  launch_gemm(p, EpiStore{}, w.stream);
  // t2 = (t1 Xt) ./ (lambda_i + theta_j)   (:172-174)
  p.M = nh; p.K = nt; p.N = nt;
  p.A = w.t1.p; p.lda = nh; p.B = w.Xt.p; p.ldb = nt; p.C = w.t2.p; p.ldc = nh;
  launch_gemm(p, EpiDivide{w.lam.p, w.theta.p}, w.stream);
  // t1 = Xs t2 ; out = t1 Xt^T   (:175)
  p.M = nh; p.K = nh; p.N = nt;
  p.A = w.Xs.p; p.lda = nh; p.B = w.t2.p; p.ldb = nh; p.C = w.t1.p; p.ldc = nh;
  launch_gemm(p, EpiStore{}, w.stream);
  p.M = nh; p.K = nt; p.N = nt;
  p.A = w.t1.p; p.lda = nh; p.B = w.XtT.p; p.ldb = nt; p.C = out; p.ldc = nh;
  launch_gemm(p, EpiStore{}, w.stream);
}

// Deterministic dot products of several (x, y) pairs, results to host.
void dots_to_host(stkg_wave& w, int count, const double* const* xs, const double* const* ys,
                  double* host_out) {
  for (int k = 0; k < count; ++k)
    dot_partials_kernel<<<kReduceBlocks, kReduceThreads, 0, w.stream>>>(
        xs[k], ys[k], w.N, w.partials.p + int64_t(k) * kReduceBlocks);
  sum_partials_kernel<<<count, kReduceThreads, 0, w.stream>>>(w.partials.p, kReduceBlocks, count,
                                                             w.scalars.p);
  STKG_CUDA_CHECK(cudaGetLastError());
  ensure_pinned(w, count);
  STKG_CUDA_CHECK(cudaMemcpyAsync(w.pinned, w.scalars.p, sizeof(double) * count,
                                  cudaMemcpyDeviceToHost, w.stream));
  STKG_CUDA_CHECK(cudaStreamSynchronize(w.stream));
  for (int k = 0; k < count; ++k) host_out[k] = w.pinned[k];
}

double norm2(stkg_wave& w, const double* x) {
  double s;
  const double* xs[1] = {x};
  dots_to_host(w, 1, xs, xs, &s);
  return std::sqrt(s);
}

// h = V(:, 0:m)^T w  (deterministic), result both on device (w.hvec) and host
void gemv_t(stkg_wave& w, int m, const double* x, double* host_h) {
  dim3 grid(kReduceBlocks, static_cast<unsigned>(ceil_div(m, kGemvCols)));
  gemv_t_kernel<<<grid, kReduceThreads, 0, w.stream>>>(w.V.p, w.N, m, x, w.partials.p);
  sum_partials_kernel<<<m, kReduceThreads, 0, w.stream>>>(w.partials.p, kReduceBlocks, m,
                                                         w.hvec.p);
  STKG_CUDA_CHECK(cudaGetLastError());
  ensure_pinned(w, m);
  STKG_CUDA_CHECK(cudaMemcpyAsync(w.pinned, w.hvec.p, sizeof(double) * m,
                                  cudaMemcpyDeviceToHost, w.stream));
  STKG_CUDA_CHECK(cudaStreamSynchronize(w.stream));
  for (int k = 0; k < m; ++k) host_h[k] = w.pinned[k];
}

void ensure_krylov(stkg_wave& w, int64_t cols, int64_t hcap) {
  if (w.v_cap < cols) {
    w.V.alloc(w.N * cols);
    w.v_cap = cols;
  }
  if (!w.w.p) {
    w.w.alloc(w.N);
    w.z.alloc(w.N);
    w.r.alloc(w.N);
    w.p.alloc(w.N);
    w.q.alloc(w.N);
    w.xk.alloc(w.N);
  }
  const size_t need = static_cast<size_t>(std::max<int64_t>(hcap, 8)) * kReduceBlocks;
  if (w.partials.n < need) w.partials.alloc(need);
  if (w.scalars.n < static_cast<size_t>(std::max<int64_t>(hcap, 8)))
    w.scalars.alloc(std::max<int64_t>(hcap, 8));
  if (w.hvec.n < static_cast<size_t>(std::max<int64_t>(hcap, 8))) w.hvec.alloc(std::max<int64_t>(hcap, 8));
}

void report_history(stkg_report* rep, double v) {
  if (!rep) return;
  if (rep->rel_res_history && rep->history_length < rep->history_capacity)
    rep->rel_res_history[rep->history_length] = v;
  rep->history_length++;
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
    }
    STKG_CUDA_CHECK(cudaStreamSynchronize(s));  // host temporaries die here
    w->partials.alloc(8 * kReduceBlocks);
    w->scalars.alloc(8);
    ensure_pinned(*w, 8);
    *out = w.release();
  });
}

int stkg_wave_destroy(stkg_wave* w) {
  return guarded([&] {
    if (!w) return;
    if (w->stream) cudaStreamSynchronize(w->stream);
    else cudaDeviceSynchronize();
    if (w->pinned) cudaFreeHost(w->pinned);
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
    precond_solve(*w, v, out);
  });
}

// gmres (stk/outer_krylov.hpp:75-164), same control flow, counters and report fields.
int stkg_gmres(stkg_wave* wv, const double* b, double* x, const stkg_gmres_config* cfg_in,
               stkg_report* rep) {
  return guarded([&] {
    STKG_REQUIRE(wv && b && x, STKG_ARGUMENT, "gmres: null argument");
    stkg_gmres_config cfg = cfg_in ? *cfg_in : stkg_gmres_config{1e-8, 200, 0, 1};
    STKG_REQUIRE(cfg.tol > 0.0 && cfg.tol < 1.0, STKG_ARGUMENT, "GmresConfig: tol must be in (0,1)");
    STKG_REQUIRE(cfg.maxit >= 1, STKG_ARGUMENT, "GmresConfig: maxit must be >= 1");
    const bool use_p = cfg.use_precond != 0;
    STKG_REQUIRE(!use_p || wv->has_precond, STKG_ARGUMENT, "gmres: no preconditioner in plan");
    stkg_wave& w = *wv;
    const auto t_start = std::chrono::steady_clock::now();
    if (rep) {
      rep->iterations = 0;
      rep->mu_mem = 0;
      rep->converged = 0;
      rep->stagnated = 0;
      rep->final_relres = 0.0;
      rep->history_length = 0;
    }
    const int cycle = cfg.restart > 0 ? cfg.restart : cfg.maxit;
    ensure_krylov(w, cycle + 1, cycle + 2);
    const int64_t N = w.N;
    STKG_CUDA_CHECK(cudaMemsetAsync(x, 0, sizeof(double) * N, w.stream));
    const double norm_b = norm2(w, b);
    bool converged = false;
    if (norm_b == 0.0) {
      if (rep) rep->converged = 1;
      return;
    }
    auto vcol = [&](int64_t j) { return w.V.p + j * N; };
    int total = 0, peak_vecs = 0;
    std::vector<double> h(cycle + 2), corr(cycle + 2);
    while (true) {
      // r = total == 0 ? b : b - apply(x)
      double* r = w.r.p;
      if (total == 0) {
        STKG_CUDA_CHECK(cudaMemcpyAsync(r, b, sizeof(double) * N, cudaMemcpyDeviceToDevice, w.stream));
      } else {
        apply_op(w, x, r);
        sub_from_kernel<<<kEwBlocks, 256, 0, w.stream>>>(b, r, N);
      }
      const double beta = norm2(w, r);
      if (beta <= cfg.tol * norm_b) {
        converged = true;
        break;
      }
      scale_copy_kernel<<<kEwBlocks, 256, 0, w.stream>>>(r, 1.0 / beta, vcol(0), N);
      std::vector<std::vector<double>> hcols;
      std::vector<double> g(cycle + 1, 0.0), cs, sn;
      g[0] = beta;
      int k = 0;
      bool done = false;
      int nbasis = 1;
      for (int j = 0; j < cycle && total < cfg.maxit; ++j, ++total) {
        // w = apply(precond(v_j))
        if (use_p) {
          precond_solve(w, vcol(j), w.z.p);
          apply_op(w, w.z.p, w.w.p);
        } else {
          apply_op(w, vcol(j), w.w.p);
        }
        const int m = j + 1;
        // Gram-Schmidt against v_0..v_j, then one re-orthogonalisation pass
        // (:111-120); run as classical GS passes (GEMV) instead of the sequential MGS loop.
        gemv_t(w, m, w.w.p, h.data());
        gemv_n_update_kernel<<<kReduceBlocks, kReduceThreads, 0, w.stream>>>(
            w.V.p, N, m, w.hvec.p, w.w.p, nullptr);
        gemv_t(w, m, w.w.p, corr.data());
        gemv_n_update_kernel<<<kReduceBlocks, kReduceThreads, 0, w.stream>>>(
            w.V.p, N, m, w.hvec.p, w.w.p, w.partials.p);
        sum_partials_kernel<<<1, kReduceThreads, 0, w.stream>>>(w.partials.p, kReduceBlocks, 1,
                                                               w.scalars.p);
        STKG_CUDA_CHECK(cudaGetLastError());
        STKG_CUDA_CHECK(cudaMemcpyAsync(w.pinned, w.scalars.p, sizeof(double),
                                        cudaMemcpyDeviceToHost, w.stream));
        STKG_CUDA_CHECK(cudaStreamSynchronize(w.stream));
        const double hlast = std::sqrt(w.pinned[0]);
        std::vector<double> col(m + 1, 0.0);
        for (int i = 0; i < m; ++i) col[i] = h[i] + corr[i];
        col[m] = hlast;
        if (!std::isfinite(hlast) || !std::isfinite(col[j]))
          throw Error(STKG_NUMERIC, "gmres: non-finite value at iteration " + std::to_string(total + 1));
        // Givens (stk/outer_krylov.hpp:37-55)
        for (int i = 0; i < j; ++i) {
          const double t = cs[i] * col[i] + sn[i] * col[i + 1];
          col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
          col[i] = t;
        }
        {
          const double a = col[j], bb = col[j + 1];
          const double rr = std::hypot(a, bb);
          const double c = rr == 0.0 ? 1.0 : a / rr;
          const double s = rr == 0.0 ? 0.0 : bb / rr;
          cs.push_back(c);
          sn.push_back(s);
          col[j] = rr;
          col[j + 1] = 0.0;
          const double t = c * g[j] + s * g[j + 1];
          g[j + 1] = -s * g[j] + c * g[j + 1];
          g[j] = t;
        }
        hcols.push_back(std::move(col));
        const double relres = std::abs(g[j + 1]) / norm_b;
        report_history(rep, relres);
        k = j + 1;
        peak_vecs = std::max(peak_vecs, nbasis + 1);
        if (relres <= cfg.tol || hlast == 0.0) {
          converged = true;
          done = true;
          ++total;
          break;
        }
        scale_copy_kernel<<<kEwBlocks, 256, 0, w.stream>>>(w.w.p, 1.0 / hlast, vcol(j + 1), N);
        ++nbasis;
      }
      if (k > 0) {
        // solve_hessenberg (stk/outer_krylov.hpp:58-67), then x += precond(sum y_i v_i)
        std::vector<double> y(k);
        for (int i = k - 1; i >= 0; --i) {
          double acc = g[i];
          for (int jj = i + 1; jj < k; ++jj) acc -= hcols[jj][i] * y[jj];
          y[i] = acc / hcols[i][i];
        }
        // xk = V y  ==  0 - V (-y)
        for (int i = 0; i < k; ++i) y[i] = -y[i];
        STKG_CUDA_CHECK(cudaMemcpyAsync(w.hvec.p, y.data(), sizeof(double) * k,
                                        cudaMemcpyHostToDevice, w.stream));
        STKG_CUDA_CHECK(cudaMemsetAsync(w.xk.p, 0, sizeof(double) * N, w.stream));
        gemv_n_update_kernel<<<kReduceBlocks, kReduceThreads, 0, w.stream>>>(
            w.V.p, N, k, w.hvec.p, w.xk.p, nullptr);
        if (use_p) {
          precond_solve(w, w.xk.p, w.z.p);
          add_kernel<<<kEwBlocks, 256, 0, w.stream>>>(w.z.p, x, N);
        } else {
          add_kernel<<<kEwBlocks, 256, 0, w.stream>>>(w.xk.p, x, N);
        }
        STKG_CUDA_CHECK(cudaStreamSynchronize(w.stream));  // y dies here
      }
      if (done || total >= cfg.maxit) break;
    }
    // final true residual (:159)
    apply_op(w, x, w.r.p);
    sub_from_kernel<<<kEwBlocks, 256, 0, w.stream>>>(b, w.r.p, N);
    const double fr = norm2(w, w.r.p) / norm_b;
    if (fr <= cfg.tol) converged = true;
    if (rep) {
      rep->iterations = total;
      rep->mu_mem = peak_vecs;
      rep->final_relres = fr;
      rep->converged = converged ? 1 : 0;
      rep->wall_time_s =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    }
  });
}

// Preconditioned conjugate gradients with TwoTermPrecond (B and P s.p.d.).
int stkg_pcg(stkg_wave* wv, const double* b, double* x, double tol, int maxit,
             stkg_report* rep) {
  return guarded([&] {
    STKG_REQUIRE(wv && b && x, STKG_ARGUMENT, "pcg: null argument");
    STKG_REQUIRE(tol > 0.0 && tol < 1.0, STKG_ARGUMENT, "pcg: tol must be in (0,1)");
    STKG_REQUIRE(maxit >= 1, STKG_ARGUMENT, "pcg: maxit must be >= 1");
    STKG_REQUIRE(wv->has_precond, STKG_ARGUMENT, "pcg: no preconditioner in plan");
    stkg_wave& w = *wv;
    const auto t_start = std::chrono::steady_clock::now();
    ensure_krylov(w, 0, 8);
    const int64_t N = w.N;
    if (rep) {
      rep->iterations = 0;
      rep->mu_mem = 5;
      rep->converged = 0;
      rep->stagnated = 0;
      rep->history_length = 0;
    }
    STKG_CUDA_CHECK(cudaMemsetAsync(x, 0, sizeof(double) * N, w.stream));
    const double norm_b = norm2(w, b);
    if (norm_b == 0.0) {
      if (rep) rep->converged = 1;
      return;
    }
    double* r = w.r.p;
    double* z = w.z.p;
    double* p = w.p.p;
    double* q = w.q.p;
    STKG_CUDA_CHECK(cudaMemcpyAsync(r, b, sizeof(double) * N, cudaMemcpyDeviceToDevice, w.stream));
    precond_solve(w, r, z);
    STKG_CUDA_CHECK(cudaMemcpyAsync(p, z, sizeof(double) * N, cudaMemcpyDeviceToDevice, w.stream));
    double rz;
    {
      const double* xs[1] = {r};
      const double* ys[1] = {z};
      dots_to_host(w, 1, xs, ys, &rz);
    }
    int it = 0;
    bool converged = false;
    while (it < maxit) {
      apply_op(w, p, q);
      double pq;
      {
        const double* xs[1] = {p};
        const double* ys[1] = {q};
        dots_to_host(w, 1, xs, ys, &pq);
      }
      if (!std::isfinite(pq) || pq <= 0.0)
        throw Error(STKG_NUMERIC, "pcg: non-positive curvature at iteration " + std::to_string(it + 1));
      const double alpha = rz / pq;
      cg_update_kernel<<<kReduceBlocks, kReduceThreads, 0, w.stream>>>(alpha, p, q, x, r, N,
                                                                      w.partials.p);
      sum_partials_kernel<<<1, kReduceThreads, 0, w.stream>>>(w.partials.p, kReduceBlocks, 1,
                                                             w.scalars.p);
      STKG_CUDA_CHECK(cudaMemcpyAsync(w.pinned, w.scalars.p, sizeof(double),
                                      cudaMemcpyDeviceToHost, w.stream));
      STKG_CUDA_CHECK(cudaStreamSynchronize(w.stream));
      ++it;
      const double relres = std::sqrt(w.pinned[0]) / norm_b;
      report_history(rep, relres);
      if (!std::isfinite(relres))
        throw Error(STKG_NUMERIC, "pcg: non-finite value at iteration " + std::to_string(it));
      if (relres <= tol) {
        converged = true;
        break;
      }
      precond_solve(w, r, z);
      double rz_new;
      {
        const double* xs[1] = {r};
        const double* ys[1] = {z};
        dots_to_host(w, 1, xs, ys, &rz_new);
      }
      const double beta = rz_new / rz;
      rz = rz_new;
      xpby_kernel<<<kEwBlocks, 256, 0, w.stream>>>(z, beta, p, N);
    }
    apply_op(w, x, w.r.p);
    sub_from_kernel<<<kEwBlocks, 256, 0, w.stream>>>(b, w.r.p, N);
    const double fr = norm2(w, w.r.p) / norm_b;
    if (rep) {
      rep->iterations = it;
      rep->final_relres = fr;
      rep->converged = (converged || fr <= tol) ? 1 : 0;
      rep->wall_time_s =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    }
  });
}

}  // extern "C"
