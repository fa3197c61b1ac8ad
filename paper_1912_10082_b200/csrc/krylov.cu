// Krylov solvers on device vectors: gmres (stk/outer_krylov.hpp:75-164) and PCG.
#include <algorithm>
#include <cstring>
#include <chrono>
#include <cmath>
#include <string>
#include <vector>

#include "krylov.cuh"

namespace stkg {
namespace {

inline unsigned ew_blocks() { return static_cast<unsigned>(num_sms()) * 8; }

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

// out[c] = sum_b partials[c * count + b], one block per column, fixed order.
__global__ void __launch_bounds__(kReduceThreads) sum_partials_kernel(
    const double* __restrict__ partials, int count, double* __restrict__ out) {
  __shared__ double red[kReduceThreads / 32];
  const int c = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < count; b += kReduceThreads) s += partials[int64_t(c) * count + b];
  s = block_sum<kReduceThreads>(s, red);
  if (threadIdx.x == 0) out[c] = s;
}

// h_c = V(:,c)^T w for c in [0, m): blockIdx.y picks 4 columns, blockIdx.x a fixed row
// slice; partials[c * gridDim.x + blockIdx.x].  V is read once (HBM-bound).
constexpr int kGemvCols = 4;
__global__ void __launch_bounds__(kReduceThreads) gemv_t_kernel(
    const double* __restrict__ V, int64_t N, int m, const double* __restrict__ w,
    double* __restrict__ partials) {
  __shared__ double red[kReduceThreads / 32];
  const int c0 = blockIdx.y * kGemvCols;
  double s[kGemvCols] = {0.0, 0.0, 0.0, 0.0};
  // kRowU rows per step: their 5 kRowU loads are independent and in flight together
  constexpr int kRowU = 4;
  const int64_t stride = int64_t(gridDim.x) * kReduceThreads;
  int64_t i = int64_t(blockIdx.x) * kReduceThreads + threadIdx.x;
  for (; i + (kRowU - 1) * stride < N; i += kRowU * stride) {
    double wi[kRowU], v[kRowU][kGemvCols];
#pragma unroll
    for (int r = 0; r < kRowU; ++r) {
      wi[r] = w[i + r * stride];
#pragma unroll
      for (int c = 0; c < kGemvCols; ++c)
        v[r][c] = c0 + c < m ? V[int64_t(c0 + c) * N + i + r * stride] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < kRowU; ++r)
#pragma unroll
      for (int c = 0; c < kGemvCols; ++c) s[c] += v[r][c] * wi[r];
  }
  for (; i < N; i += stride) {
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

// w -= V h (h on the device, m columns); optionally ||w||^2 partials.
__global__ void __launch_bounds__(kReduceThreads) gemv_n_update_kernel(
    const double* __restrict__ V, int64_t N, int m, const double* __restrict__ h,
    double* __restrict__ w, double* __restrict__ partials) {
  __shared__ double red[kReduceThreads / 32];
  double nrm = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kReduceThreads + threadIdx.x; i < N;
       i += int64_t(gridDim.x) * kReduceThreads) {
    double acc = w[i];
    int c = 0;
    // 8 columns per step: 8 independent loads in flight per thread
    for (; c + 8 <= m; c += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = V[int64_t(c + q) * N + i];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc -= h[c + q] * v[q];
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

__global__ void sub_from_kernel(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    y[i] = x[i] - y[i];
}

__global__ void add_kernel(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    y[i] += x[i];
}

void report_history(stkg_report* rep, double v) {
  if (!rep) return;
  if (rep->rel_res_history && rep->history_length < rep->history_capacity)
    rep->rel_res_history[rep->history_length] = v;
  rep->history_length++;
}

// scalars -> host (synchronous)
void fetch(Krylov& k, int count, double* out) {
  k.pin(count);
  STKG_CUDA_CHECK(cudaMemcpyAsync(k.pinned, k.scalars.p, sizeof(double) * count,
                                  cudaMemcpyDeviceToHost, k.stream));
  STKG_CUDA_CHECK(cudaStreamSynchronize(k.stream));
  for (int i = 0; i < count; ++i) out[i] = k.pinned[i];
}

// h = V(:, 0:m)^T x into the device vector out (no host round trip)
void gemv_t_dev(Krylov& k, int m, const double* x, double* out) {
  dim3 grid(kReduceBlocks, static_cast<unsigned>(ceil_div(m, kGemvCols)));
  gemv_t_kernel<<<grid, kReduceThreads, 0, k.stream>>>(k.V.p, k.N, m, x, k.partials.p);
  sum_partials_kernel<<<m, kReduceThreads, 0, k.stream>>>(k.partials.p, kReduceBlocks, out);
  STKG_CUDA_CHECK(cudaGetLastError());
}


}  // namespace

Krylov::~Krylov() {
  if (pinned) cudaFreeHost(pinned);
}

void Krylov::pin(int count) {
  if (count <= pinned_cap) return;
  if (pinned) cudaFreeHost(pinned);
  pinned = nullptr;
  STKG_CUDA_CHECK(cudaMallocHost(&pinned, sizeof(double) * count));
  pinned_cap = count;
}

void Krylov::ensure(int64_t cols, int64_t hcap) {
  if (v_cap < cols) {
    V.alloc(N * cols);
    v_cap = cols;
  }
  if (!w.p) {
    w.alloc(N);
    z.alloc(N);
    r.alloc(N);
    p.alloc(N);
    q.alloc(N);
    xk.alloc(N);
  }
  const int64_t h = std::max<int64_t>(hcap, 8);
  if (partials.n < static_cast<size_t>(h * kReduceBlocks)) partials.alloc(h * kReduceBlocks);
  if (scalars.n < static_cast<size_t>(h)) scalars.alloc(h);
  if (hvec.n < static_cast<size_t>(2 * h)) hvec.alloc(2 * h);  // two Gram-Schmidt passes
  pin(static_cast<int>(2 * h + 1));  // once: cudaMallocHost synchronises the device
}

double kdot(Krylov& k, const double* x, const double* y) {
  dot_partials_kernel<<<kReduceBlocks, kReduceThreads, 0, k.stream>>>(x, y, k.N, k.partials.p);
  sum_partials_kernel<<<1, kReduceThreads, 0, k.stream>>>(k.partials.p, kReduceBlocks, k.scalars.p);
  STKG_CUDA_CHECK(cudaGetLastError());
  double s;
  fetch(k, 1, &s);
  return s;
}

double knorm(Krylov& k, const double* x) { return std::sqrt(kdot(k, x, x)); }

void gmres_run(Krylov& k, const DevOp& apply, const DevOp* precond, const double* b, double* x,
               const stkg_gmres_config& cfg, stkg_report* rep) {
  STKG_REQUIRE(cfg.tol > 0.0 && cfg.tol < 1.0, STKG_ARGUMENT, "GmresConfig: tol must be in (0,1)");
  STKG_REQUIRE(cfg.maxit >= 1, STKG_ARGUMENT, "GmresConfig: maxit must be >= 1");
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
  k.ensure(int64_t(cycle) + 1, int64_t(cycle) + 2);
  const int64_t N = k.N;
  cudaStream_t s = k.stream;
  STKG_CUDA_CHECK(cudaMemsetAsync(x, 0, sizeof(double) * N, s));
  const double norm_b = knorm(k, b);
  if (norm_b == 0.0) {
    if (rep) rep->converged = 1;
    return;
  }
  auto vcol = [&](int64_t j) { return k.V.p + j * N; };
  bool converged = false;
  int total = 0, peak_vecs = 0;
  std::vector<double> h(cycle + 2), corr(cycle + 2);
  while (true) {
    double* r = k.r.p;
    if (total == 0) {
      STKG_CUDA_CHECK(cudaMemcpyAsync(r, b, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    } else {
      apply(x, r);
      sub_from_kernel<<<ew_blocks(), 256, 0, s>>>(b, r, N);
    }
    const double beta = knorm(k, r);
    if (beta <= cfg.tol * norm_b) {
      converged = true;
      break;
    }
    scale_copy_kernel<<<ew_blocks(), 256, 0, s>>>(r, 1.0 / beta, vcol(0), N);
    std::vector<std::vector<double>> hcols;
    std::vector<double> g(cycle + 1, 0.0), cs, sn;
    g[0] = beta;
    int kdim = 0, nbasis = 1;
    bool done = false;
    for (int j = 0; j < cycle && total < cfg.maxit; ++j, ++total) {
      if (precond) {
        (*precond)(vcol(j), k.z.p);
        apply(k.z.p, k.w.p);
      } else {
        apply(vcol(j), k.w.p);
      }
      const int m = j + 1;
      // both Gram-Schmidt passes stay on the device (h1 in hvec[0:m), h2 in hvec[hoff:hoff+m));
      // one host round trip per iteration fetches h1, h2 and ||w||^2 together
      const int64_t hoff = k.hvec.n / 2;
      double* h1d = k.hvec.p;
      double* h2d = k.hvec.p + hoff;
      gemv_t_dev(k, m, k.w.p, h1d);  // (:111-115)
      gemv_n_update_kernel<<<kReduceBlocks, kReduceThreads, 0, s>>>(k.V.p, N, m, h1d, k.w.p,
                                                                   nullptr);
      gemv_t_dev(k, m, k.w.p, h2d);  // re-orthogonalisation (:116-120)
      gemv_n_update_kernel<<<kReduceBlocks, kReduceThreads, 0, s>>>(k.V.p, N, m, h2d, k.w.p,
                                                                   k.partials.p);
      sum_partials_kernel<<<1, kReduceThreads, 0, s>>>(k.partials.p, kReduceBlocks, k.scalars.p);
      STKG_CUDA_CHECK(cudaGetLastError());
      k.pin(2 * m + 1);
      STKG_CUDA_CHECK(cudaMemcpyAsync(k.pinned, h1d, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
      STKG_CUDA_CHECK(cudaMemcpyAsync(k.pinned + m, h2d, sizeof(double) * m,
                                      cudaMemcpyDeviceToHost, s));
      STKG_CUDA_CHECK(cudaMemcpyAsync(k.pinned + 2 * m, k.scalars.p, sizeof(double),
                                      cudaMemcpyDeviceToHost, s));
      STKG_CUDA_CHECK(cudaStreamSynchronize(s));
      for (int i = 0; i < m; ++i) {
        h[i] = k.pinned[i];
        corr[i] = k.pinned[m + i];
      }
      const double h2 = k.pinned[2 * m];
      const double hlast = std::sqrt(h2);
      std::vector<double> col(m + 1, 0.0);
      for (int i = 0; i < m; ++i) col[i] = h[i] + corr[i];
      col[m] = hlast;
      if (!std::isfinite(hlast) || !std::isfinite(col[j]))
        throw Error(STKG_NUMERIC, "gmres: non-finite value at iteration " + std::to_string(total + 1));
      // Givens least squares (stk/outer_krylov.hpp:37-55)
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * col[i] + sn[i] * col[i + 1];
        col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
        col[i] = t;
      }
      {
        const double a = col[j], bb = col[j + 1];
        const double rr = std::hypot(a, bb);
        const double c = rr == 0.0 ? 1.0 : a / rr;
        const double sv = rr == 0.0 ? 0.0 : bb / rr;
        cs.push_back(c);
        sn.push_back(sv);
        col[j] = rr;
        col[j + 1] = 0.0;
        const double t = c * g[j] + sv * g[j + 1];
        g[j + 1] = -sv * g[j] + c * g[j + 1];
        g[j] = t;
      }
      hcols.push_back(std::move(col));
      const double relres = std::abs(g[j + 1]) / norm_b;
      report_history(rep, relres);
      kdim = j + 1;
      peak_vecs = std::max(peak_vecs, nbasis + 1);
      if (relres <= cfg.tol || hlast == 0.0) {
        converged = true;
        done = true;
        ++total;
        break;
      }
      scale_copy_kernel<<<ew_blocks(), 256, 0, s>>>(k.w.p, 1.0 / hlast, vcol(j + 1), N);
      ++nbasis;
    }
    if (kdim > 0) {
      // solve_hessenberg (stk/outer_krylov.hpp:58-67); x += precond(V y)
      std::vector<double> y(kdim);
      for (int i = kdim - 1; i >= 0; --i) {
        double acc = g[i];
        for (int jj = i + 1; jj < kdim; ++jj) acc -= hcols[jj][i] * y[jj];
        y[i] = acc / hcols[i][i];
      }
      for (int i = 0; i < kdim; ++i) y[i] = -y[i];  // xk = 0 - V(-y)
      STKG_CUDA_CHECK(cudaMemcpyAsync(k.hvec.p, y.data(), sizeof(double) * kdim,
                                      cudaMemcpyHostToDevice, s));
      STKG_CUDA_CHECK(cudaMemsetAsync(k.xk.p, 0, sizeof(double) * N, s));
      gemv_n_update_kernel<<<kReduceBlocks, kReduceThreads, 0, s>>>(k.V.p, N, kdim, k.hvec.p,
                                                                   k.xk.p, nullptr);
      if (precond) {
        (*precond)(k.xk.p, k.z.p);
        add_kernel<<<ew_blocks(), 256, 0, s>>>(k.z.p, x, N);
      } else {
        add_kernel<<<ew_blocks(), 256, 0, s>>>(k.xk.p, x, N);
      }
      STKG_CUDA_CHECK(cudaStreamSynchronize(s));  // y dies here
    }
    if (done || total >= cfg.maxit) break;
  }
  apply(x, k.r.p);  // final true residual (:159)
  sub_from_kernel<<<ew_blocks(), 256, 0, s>>>(b, k.r.p, N);
  const double fr = knorm(k, k.r.p) / norm_b;
  if (fr <= cfg.tol) converged = true;
  if (rep) {
    rep->iterations = total;
    rep->mu_mem = peak_vecs;
    rep->final_relres = fr;
    rep->converged = converged ? 1 : 0;
    rep->wall_time_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  }
}

namespace {

// PCG scalars live on the device so that an iteration needs no host round trip; the host
// only polls `done` every kPcgChunk iterations.
struct PcgState {
  double rz, pq, alpha, beta, normb, tol;
  double rel_prev, rel_last;  // the last two relative residuals (sizing the next chunk)
  int done, iters, error, maxit;
};
constexpr int kPcgChunk = 8;

__device__ double sum_fixed(const double* partials, int count, double* red) {
  double s = 0.0;
  for (int b = threadIdx.x; b < count; b += kReduceThreads) s += partials[b];
  return block_sum<kReduceThreads>(s, red);
}

__global__ void __launch_bounds__(kReduceThreads) pcg_init_kernel(const double* partials_rz,
                                                                  PcgState* st, double normb,
                                                                  double tol, int maxit) {
  __shared__ double red[kReduceThreads / 32];
  const double rz = sum_fixed(partials_rz, kReduceBlocks, red);
  if (threadIdx.x == 0) {
    st->rz = rz;
    st->normb = normb;
    st->tol = tol;
    st->maxit = maxit;
    st->done = 0;
    st->iters = 0;
    st->error = 0;
    st->rel_prev = st->rel_last = 1.0;
  }
}

__global__ void __launch_bounds__(kReduceThreads) pcg_alpha_kernel(const double* partials,
                                                                   PcgState* st) {
  __shared__ double red[kReduceThreads / 32];
  if (st->done) return;
  const double pq = sum_fixed(partials, kReduceBlocks, red);
  if (threadIdx.x == 0) {
    st->pq = pq;
    if (!(pq > 0.0) || !isfinite(pq)) {
      st->error = 1;
      st->done = 1;
    } else {
      st->alpha = st->rz / pq;
    }
  }
}

__global__ void __launch_bounds__(kReduceThreads) pcg_update_kernel(
    const PcgState* st, const double* __restrict__ p, const double* __restrict__ q,
    double* __restrict__ x, double* __restrict__ r, int64_t n, double* __restrict__ partials) {
  __shared__ double red[kReduceThreads / 32];
  if (st->done) return;
  const double a = st->alpha;
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

__global__ void __launch_bounds__(kReduceThreads) pcg_check_kernel(const double* partials,
                                                                   PcgState* st, double* hist) {
  __shared__ double red[kReduceThreads / 32];
  if (st->done) return;
  const double r2 = sum_fixed(partials, kReduceBlocks, red);
  if (threadIdx.x == 0) {
    const double relres = sqrt(r2) / st->normb;
    hist[st->iters] = relres;
    st->rel_prev = st->rel_last;
    st->rel_last = relres;
    st->iters += 1;
    if (!isfinite(relres)) {
      st->error = 2;
      st->done = 1;
    } else if (relres <= st->tol || st->iters >= st->maxit) {
      st->done = 1;
    }
  }
}

__global__ void __launch_bounds__(kReduceThreads) pcg_dot_kernel(
    const PcgState* st, const double* __restrict__ x, const double* __restrict__ y, int64_t n,
    double* __restrict__ partials) {
  __shared__ double red[kReduceThreads / 32];
  if (st->done) return;
  double s = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kReduceThreads + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * kReduceThreads)
    s += x[i] * y[i];
  s = block_sum<kReduceThreads>(s, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kReduceThreads) pcg_beta_kernel(const double* partials,
                                                                  PcgState* st) {
  __shared__ double red[kReduceThreads / 32];
  if (st->done) return;
  const double rz_new = sum_fixed(partials, kReduceBlocks, red);
  if (threadIdx.x == 0) {
    st->beta = rz_new / st->rz;
    st->rz = rz_new;
  }
}

__global__ void pcg_xpby_kernel(const PcgState* st, const double* __restrict__ z,
                                double* __restrict__ p, int64_t n) {
  if (st->done) return;
  const double b = st->beta;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = z[i] + b * p[i];
}

}  // namespace

void pcg_run(Krylov& k, const DevOp& apply, const DevOp& precond, const double* b, double* x,
             double tol, int maxit, stkg_report* rep) {
  STKG_REQUIRE(tol > 0.0 && tol < 1.0, STKG_ARGUMENT, "pcg: tol must be in (0,1)");
  STKG_REQUIRE(maxit >= 1, STKG_ARGUMENT, "pcg: maxit must be >= 1");
  const auto t_start = std::chrono::steady_clock::now();
  k.ensure(0, 8);
  const int64_t N = k.N;
  cudaStream_t s = k.stream;
  if (rep) {
    rep->iterations = 0;
    rep->mu_mem = 5;
    rep->converged = 0;
    rep->stagnated = 0;
    rep->history_length = 0;
  }
  STKG_CUDA_CHECK(cudaMemsetAsync(x, 0, sizeof(double) * N, s));
  const double norm_b = knorm(k, b);
  if (norm_b == 0.0) {
    if (rep) rep->converged = 1;
    return;
  }
  if (k.state_buf.n < (sizeof(PcgState) + 7) / 8) k.state_buf.alloc((sizeof(PcgState) + 7) / 8);
  if (k.hist_buf.n < static_cast<size_t>(maxit)) k.hist_buf.alloc(maxit);
  PcgState* st = reinterpret_cast<PcgState*>(k.state_buf.p);
  double* hist = k.hist_buf.p;
  double *r = k.r.p, *z = k.z.p, *p = k.p.p, *q = k.q.p;
  STKG_CUDA_CHECK(cudaMemcpyAsync(r, b, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
  precond(r, z);
  STKG_CUDA_CHECK(cudaMemcpyAsync(p, z, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
  dot_partials_kernel<<<kReduceBlocks, kReduceThreads, 0, s>>>(r, z, N, k.partials.p);
  pcg_init_kernel<<<1, kReduceThreads, 0, s>>>(k.partials.p, st, norm_b, tol, maxit);
  STKG_CUDA_CHECK(cudaGetLastError());
  k.skip = &st->done;  // library operators turn into no-ops once the device test fires
  struct SkipReset {  // cleared on every exit path, including a throw inside the loop
    const int*& ref;
    ~SkipReset() { ref = nullptr; }
  } skip_reset{k.skip};
  PcgState hs{};
  k.pin(sizeof(PcgState) / 8 + 1);
  int enqueued = 0;
  int chunk = kPcgChunk;
  while (true) {
    for (int c = 0; c < chunk && enqueued < maxit; ++c, ++enqueued) {
      apply(p, q);
      pcg_dot_kernel<<<kReduceBlocks, kReduceThreads, 0, s>>>(st, p, q, N, k.partials.p);
      pcg_alpha_kernel<<<1, kReduceThreads, 0, s>>>(k.partials.p, st);
      pcg_update_kernel<<<kReduceBlocks, kReduceThreads, 0, s>>>(st, p, q, x, r, N, k.partials.p);
      pcg_check_kernel<<<1, kReduceThreads, 0, s>>>(k.partials.p, st, hist);
      precond(r, z);
      pcg_dot_kernel<<<kReduceBlocks, kReduceThreads, 0, s>>>(st, r, z, N, k.partials.p);
      pcg_beta_kernel<<<1, kReduceThreads, 0, s>>>(k.partials.p, st);
      pcg_xpby_kernel<<<ew_blocks(), 256, 0, s>>>(st, z, p, N);
    }
    STKG_CUDA_CHECK(cudaGetLastError());
    STKG_CUDA_CHECK(cudaMemcpyAsync(k.pinned, st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    STKG_CUDA_CHECK(cudaStreamSynchronize(s));
    std::memcpy(&hs, k.pinned, sizeof(PcgState));
    if (hs.done || enqueued >= maxit) break;
    // size the next chunk from the observed contraction (iterations past convergence still
    // launch their kernels, as no-ops): a rapidly converging preconditioner (the modal banded
    // one needs ~9 iterations) otherwise pays up to kPcgChunk - 1 wasted iterations
    chunk = kPcgChunk;
    if (hs.iters >= 2 && hs.rel_prev > 0.0 && hs.rel_last > 0.0 && hs.rel_last < hs.rel_prev) {
      const double rho = hs.rel_last / hs.rel_prev;
      const double need = std::log(tol / hs.rel_last) / std::log(rho);
      if (need > 0.0 && need < kPcgChunk) chunk = std::max(1, static_cast<int>(std::ceil(need)) + 1);
    }
  }
  k.skip = nullptr;  // the true-residual apply below must run
  if (hs.error == 1)
    throw Error(STKG_NUMERIC, "pcg: non-positive curvature at iteration " + std::to_string(hs.iters + 1));
  if (hs.error == 2)
    throw Error(STKG_NUMERIC, "pcg: non-finite value at iteration " + std::to_string(hs.iters));
  const int it = hs.iters;
  std::vector<double> h(static_cast<size_t>(it));
  if (it > 0)
    STKG_CUDA_CHECK(cudaMemcpy(h.data(), hist, sizeof(double) * it, cudaMemcpyDeviceToHost));
  for (int i = 0; i < it; ++i) report_history(rep, h[i]);
  const bool converged = it > 0 && h[it - 1] <= tol;
  apply(x, k.r.p);  // true final residual
  sub_from_kernel<<<ew_blocks(), 256, 0, s>>>(b, k.r.p, N);
  const double fr = knorm(k, k.r.p) / norm_b;
  if (rep) {
    rep->iterations = it;
    rep->final_relres = fr;
    rep->converged = (converged || fr <= tol) ? 1 : 0;
    rep->wall_time_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  }
}

}  // namespace stkg

using namespace stkg;

namespace {
DevOp wrap(stkg_vec_op op, void* user, cudaStream_t s) {
  return [=](const double* x, double* y) {
    const int st = op(user, x, y, s);
    if (st != STKG_OK)
      throw Error(st, "operator callback failed with status " + std::to_string(st));
  };
}
}  // namespace

extern "C" {

int stkg_gmres_op(int64_t n, stkg_vec_op apply, void* apply_user, stkg_vec_op precond,
                  void* precond_user, const double* b, double* x, const stkg_gmres_config* cfg,
                  stkg_report* report, void* cuda_stream) {
  return guarded([&] {
    STKG_REQUIRE(n >= 1 && apply && b && x, STKG_ARGUMENT, "gmres: bad arguments");
    Krylov k;
    k.N = n;
    k.stream = static_cast<cudaStream_t>(cuda_stream);
    const DevOp a = wrap(apply, apply_user, k.stream);
    const DevOp p = precond ? wrap(precond, precond_user, k.stream) : DevOp();
    const stkg_gmres_config c = cfg ? *cfg : stkg_gmres_config{1e-8, 200, 0, 1};
    gmres_run(k, a, precond ? &p : nullptr, b, x, c, report);
    STKG_CUDA_CHECK(cudaStreamSynchronize(k.stream));
  });
}

int stkg_pcg_op(int64_t n, stkg_vec_op apply, void* apply_user, stkg_vec_op precond,
                void* precond_user, const double* b, double* x, double tol, int maxit,
                stkg_report* report, void* cuda_stream) {
  return guarded([&] {
    STKG_REQUIRE(n >= 1 && apply && precond && b && x, STKG_ARGUMENT, "pcg: bad arguments");
    Krylov k;
    k.N = n;
    k.stream = static_cast<cudaStream_t>(cuda_stream);
    pcg_run(k, wrap(apply, apply_user, k.stream), wrap(precond, precond_user, k.stream), b, x,
            tol, maxit, report);
    STKG_CUDA_CHECK(cudaStreamSynchronize(k.stream));
  });
}

}  // extern "C"
