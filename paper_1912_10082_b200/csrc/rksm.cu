// Rational Krylov subspace method for the heat system (north_star item 3):
// rksm_solve (stk/rksm.hpp:127-234), the paper's own solver for low-rank loads F = L R^T.
//
// Device building blocks (n_x-long blocks of b columns):
//   * shifted solves (A - sigma M)^-1 M W: batched tridiagonal (Thomas) solves in 1D, and in
//     the tensor eigenbasis X (Lambda - sigma)^-1 X^T M W (dense backend) or
//     S (Lambda - sigma)^-1 S W (P1 fast-sine backend) in 2D/3D -- exact, no factorisation;
//   * block Gram-Schmidt as tall-skinny GEMMs: H = V^T W (one pass over V, deterministic
//     fixed-grid reduction) and W -= V H (one pass), applied twice (stk/rksm.hpp:213);
//   * projections V^T M V, V^T A V (:180-183), grown by the new block only;
//   * rank-revealing orthonormalisation (ColPivHouseholderQR in the reference, :146-151,
//     :214-224) as pivoted Cholesky-QR2 (Gram on the device, pivoted Cholesky on the host);
//   * the factored residual (residual_norm_factored, stk/sylvester.hpp:69-85): the left
//     factors [F1, M V, A V] are orthonormalised incrementally into Q_res, so
//     ||F - B(U)||_F = ||Q_res^T [F1, MV, AV] W^T||_F with a small host product.
// Host: the k x k pencil eigenproblem, the projected heat solve, the adaptive poles
// (adaptive_next_shift, stk/rksm.hpp:67-102), Givens-free bookkeeping and the final
// truncation (lowrank_truncate, stk/la_core.hpp:134-162, via one-sided Jacobi SVD).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <limits>
#include <string>
#include <vector>

#include "common.cuh"
#include "gemm_f64.cuh"
#include "heat_plan.cuh"
#include "hostla.hpp"

using namespace stkg;

namespace {

constexpr int kTsCols = 4;   // V columns per block in the tall-skinny Gram
constexpr int kTsRhs = 8;    // W columns per pass
inline unsigned ew_blocks() { return static_cast<unsigned>(num_sms()) * 8; }

// Tall-skinny Gram V(:, c0 + 0..k)^T W(:, 0..b): CTA (g, cb) covers rows of slab g (of
// gridDim.x slabs) and the 32 V columns of block cb, each warp 4 columns; lanes stride the
// rows.  The 8 warps read the same W rows, so W crosses L2 once per column block (not once
// per 4 columns).  Partials [(j k + c) gridDim.x + g] are summed in index order by
// reduce_rows_kernel: deterministic for given sizes.
template <int B>
__global__ void __launch_bounds__(256) ts_gram_kernel(const double* __restrict__ V, int64_t n,
                                                      int k, const double* __restrict__ W,
                                                      int b, double* __restrict__ partials) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c0 = blockIdx.y * (8 * kTsCols) + warp * kTsCols;
  const int64_t rows = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = int64_t(blockIdx.x) * rows;
  const int64_t r1 = r0 + rows < n ? r0 + rows : n;
  double s[kTsCols][B];
#pragma unroll
  for (int c = 0; c < kTsCols; ++c)
#pragma unroll
    for (int j = 0; j < B; ++j) s[c][j] = 0.0;
  if (c0 < k) {
    for (int64_t i = r0 + lane; i < r1; i += 32) {
      double w[B];
#pragma unroll
      for (int j = 0; j < B; ++j) w[j] = j < b ? W[int64_t(j) * n + i] : 0.0;
#pragma unroll
      for (int c = 0; c < kTsCols; ++c) {
        if (c0 + c < k) {
          const double v = V[int64_t(c0 + c) * n + i];
#pragma unroll
          for (int j = 0; j < B; ++j) s[c][j] = fma(v, w[j], s[c][j]);
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kTsCols; ++c)
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const double t = warp_sum(s[c][j]);
      if (lane == 0 && c0 + c < k && j < b)
        partials[(int64_t(j) * k + c0 + c) * gridDim.x + blockIdx.x] = t;
    }
}

// Row r = j * kk + c of the partials -> out[j * ld + c] (a kk x bb block of a column-major
// matrix with leading dimension ld).
__global__ void __launch_bounds__(256) reduce_rows_kernel(const double* __restrict__ partials,
                                                          int count, int kk, int64_t ld,
                                                          double* __restrict__ out) {
  __shared__ double red[8];
  double s = 0.0;
  for (int b = threadIdx.x; b < count; b += 256) s += partials[int64_t(blockIdx.x) * count + b];
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) out[int64_t(blockIdx.x / kk) * ld + blockIdx.x % kk] = s;
}

// W (n x b) -= V (n x k) H (k x b, column-major, staged in shared memory)
template <int B>
__global__ void __launch_bounds__(256) ts_update_kernel(double* __restrict__ W, int64_t n, int b,
                                                        const double* __restrict__ V, int k,
                                                        const double* __restrict__ H) {
  extern __shared__ double hs[];
  for (int e = threadIdx.x; e < k * B; e += 256) hs[e] = e < k * b ? H[e] : 0.0;  // pad to B
  __syncthreads();
  for (int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x; i < n; i += int64_t(gridDim.x) * 256) {
    double acc[B];
#pragma unroll
    for (int j = 0; j < B; ++j) acc[j] = j < b ? W[int64_t(j) * n + i] : 0.0;
    for (int c = 0; c < k; ++c) {
      const double v = V[int64_t(c) * n + i];
#pragma unroll
      for (int j = 0; j < B; ++j) acc[j] -= v * hs[j * k + c];
    }
#pragma unroll
    for (int j = 0; j < B; ++j)
      if (j < b) W[int64_t(j) * n + i] = acc[j];
  }
}

__global__ void scale_kernel(double* __restrict__ x, int64_t n, double alpha) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    x[i] *= alpha;
}

__global__ void scale_modes_kernel(double* __restrict__ Y, int64_t nx, int cols, ModeLambda lam,
                                   double sigma) {
  const int64_t total = nx * cols;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x)
    Y[e] /= (lam(e % nx) - sigma);
}

// Batched tridiagonal solves (A - sigma M) x = r, one column per thread (Thomas algorithm;
// A - sigma M is s.p.d. for sigma < 0, so no pivoting is needed).  X holds r on entry.
__global__ void thomas_kernel(const double* __restrict__ md, const double* __restrict__ mo,
                              const double* __restrict__ ad, const double* __restrict__ ao,
                              int64_t n, double sigma, double* __restrict__ X, int cols,
                              double* __restrict__ cp) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  double* x = X + int64_t(c) * n;
  double* cpc = cp + int64_t(c) * n;
  double diag = ad[0] - sigma * md[0];
  double sup = n > 1 ? ao[0] - sigma * mo[0] : 0.0;
  cpc[0] = sup / diag;
  x[0] = x[0] / diag;
  for (int64_t i = 1; i < n; ++i) {
    const double sub = ao[i - 1] - sigma * mo[i - 1];
    diag = ad[i] - sigma * md[i];
    const double m = diag - sub * cpc[i - 1];
    sup = i + 1 < n ? ao[i] - sigma * mo[i] : 0.0;
    cpc[i] = sup / m;
    x[i] = (x[i] - sub * x[i - 1]) / m;
  }
  for (int64_t i = n - 2; i >= 0; --i) x[i] -= cpc[i] * x[i + 1];
}

// Growable device block of n-long columns.
struct Block {
  int64_t n = 0;
  int64_t cols = 0;
  DevBuf buf;
  double* col(int64_t c) { return buf.p + c * n; }
  void reserve(int64_t need, cudaStream_t s) {
    if (static_cast<int64_t>(buf.n) >= need * n) return;
    int64_t cap = std::max<int64_t>(need, 2 * static_cast<int64_t>(buf.n / std::max<int64_t>(n, 1)));
    DevBuf nb(static_cast<size_t>(cap * n));
    if (cols > 0)
      STKG_CUDA_CHECK(cudaMemcpyAsync(nb.p, buf.p, sizeof(double) * cols * n,
                                      cudaMemcpyDeviceToDevice, s));
    STKG_CUDA_CHECK(cudaStreamSynchronize(s));
    std::swap(buf.p, nb.p);
    std::swap(buf.n, nb.n);
  }
};

class Rksm {
 public:
  Rksm(stkg_heat& h, const stkg_rksm_options& o)
      : h_(h), o_(o), n_(h.nx), nt_(h.nt), partials_(h.rk_partials), hdev_(h.rk_hdev),
        ones_(h.rk_ones), zeros_(h.rk_zeros), slots_(h.rk_slots), hpin_(h.rk_pin),
        hpin_n_(h.rk_pin_n) {
    s_ = h.stream;
    if (!partials_.p) {  // first use of this plan: fixed buffers
      partials_.alloc(static_cast<size_t>(kReduceBlocks) * 16 * 1024);
      hdev_.alloc(16 * 1024);
      ones_.alloc(kTsRhs * 2);
      zeros_.alloc(kTsRhs * 2);
      std::vector<double> one(kTsRhs * 2, 1.0), zero(kTsRhs * 2, 0.0);
      ones_.upload(one.data(), one.size(), s_);
      zeros_.upload(zero.data(), zero.size(), s_);
      STKG_CUDA_CHECK(cudaStreamSynchronize(s_));
    }
  }

  // ------------------------------------------------------------- device helpers ----
  // Growable per-purpose device scratch (no cudaMalloc inside the iteration once warm).
  double* scratch(int slot, size_t count) {
    DevBuf& b = slots_[slot];
    if (b.n < count) {
      STKG_CUDA_CHECK(cudaStreamSynchronize(s_));
      b.alloc(std::max(count, 2 * b.n));
    }
    return b.p;
  }
  double* pinned(size_t count) {
    if (hpin_n_ < count) {
      STKG_CUDA_CHECK(cudaStreamSynchronize(s_));
      if (hpin_) cudaFreeHost(hpin_);
      hpin_n_ = std::max(count, 2 * hpin_n_);
      STKG_CUDA_CHECK(cudaMallocHost(&hpin_, sizeof(double) * hpin_n_));
    }
    return hpin_;
  }

  // Hd (k x b, column-major, device, ld k) = V(:, 0:k)^T W(:, 0:b); asynchronous,
  // deterministic (fixed-grid partials summed in index order).
  void gram_dev(const double* V, int64_t k, const double* W, int64_t b, double* Hd) {
    for (int64_t j0 = 0; j0 < b; j0 += kTsRhs) {
      const int bb = static_cast<int>(std::min<int64_t>(kTsRhs, b - j0));
      for (int64_t c0 = 0; c0 < k; c0 += 1024) {
        const int kk = static_cast<int>(std::min<int64_t>(1024, k - c0));
        const int cblocks = static_cast<int>(ceil_div(kk, 8 * kTsCols));
        const int slabs = static_cast<int>(std::max<int64_t>(
            16, std::min<int64_t>(kReduceBlocks, 2 * kReduceBlocks / cblocks)));
        dim3 grid(static_cast<unsigned>(slabs), static_cast<unsigned>(cblocks));
        ts_gram_kernel<kTsRhs><<<grid, 256, 0, s_>>>(V + c0 * n_, n_, kk, W + j0 * n_, bb,
                                                     partials_.p);
        reduce_rows_kernel<<<kk * bb, 256, 0, s_>>>(partials_.p, slabs, kk, k,
                                                    Hd + j0 * k + c0);
        STKG_CUDA_CHECK(cudaGetLastError());
      }
    }
  }

  // H (k x b, column-major, host) = V(:, 0:k)^T W(:, 0:b): one device->host read.
  hla::Mat gram(const double* V, int64_t k, const double* W, int64_t b) {
    hla::Mat H(static_cast<size_t>(k * b));
    if (k == 0 || b == 0) return H;
    double* hd = scratch(kSlotGram, H.size());
    gram_dev(V, k, W, b, hd);
    double* hp = pinned(H.size());
    STKG_CUDA_CHECK(cudaMemcpyAsync(hp, hd, sizeof(double) * H.size(), cudaMemcpyDeviceToHost, s_));
    STKG_CUDA_CHECK(cudaStreamSynchronize(s_));
    std::copy(hp, hp + H.size(), H.begin());
    return H;
  }

  // Several Grams with one device->host read: gram_batch({{V, k, W, b}, ...}).
  struct GramReq {
    const double* V;
    int64_t k;
    const double* W;
    int64_t b;
  };
  std::vector<hla::Mat> gram_batch(const std::vector<GramReq>& reqs) {
    size_t total = 0;
    for (const auto& r : reqs) total += static_cast<size_t>(r.k * r.b);
    std::vector<hla::Mat> out(reqs.size());
    if (total == 0) {
      for (size_t q = 0; q < reqs.size(); ++q) out[q].assign(static_cast<size_t>(reqs[q].k * reqs[q].b), 0.0);
      return out;
    }
    double* hd = scratch(kSlotGram, total);
    size_t off = 0;
    for (const auto& r : reqs) {
      if (r.k > 0 && r.b > 0) gram_dev(r.V, r.k, r.W, r.b, hd + off);
      off += static_cast<size_t>(r.k * r.b);
    }
    double* hp = pinned(total);
    STKG_CUDA_CHECK(cudaMemcpyAsync(hp, hd, sizeof(double) * total, cudaMemcpyDeviceToHost, s_));
    STKG_CUDA_CHECK(cudaStreamSynchronize(s_));
    off = 0;
    for (size_t q = 0; q < reqs.size(); ++q) {
      const size_t n = static_cast<size_t>(reqs[q].k * reqs[q].b);
      out[q].assign(hp + off, hp + off + n);
      off += n;
    }
    return out;
  }

  // W(:, 0:b) -= V(:, 0:k) Hd (k x b, device, ld k); asynchronous.
  void update_dev(double* W, int64_t b, const double* V, int64_t k, const double* Hd) {
    if (k == 0 || b == 0) return;
    static const bool configured = [] {
      STKG_CUDA_CHECK(cudaFuncSetAttribute(ts_update_kernel<kTsRhs>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      return true;
    }();
    (void)configured;
    const size_t smem = sizeof(double) * static_cast<size_t>(k) * kTsRhs;
    STKG_REQUIRE(smem <= 200 * 1024, STKG_ARGUMENT, "rksm: Krylov basis too large");
    for (int64_t j0 = 0; j0 < b; j0 += kTsRhs) {
      const int bb = static_cast<int>(std::min<int64_t>(kTsRhs, b - j0));
      ts_update_kernel<kTsRhs><<<ew_blocks(), 256, smem, s_>>>(W + j0 * n_, n_, bb, V, static_cast<int>(k),
                                                       Hd + j0 * k);
      STKG_CUDA_CHECK(cudaGetLastError());
    }
  }

  // W(:, 0:b) -= V(:, 0:k) H (k x b host)
  void update(double* W, int64_t b, const double* V, int64_t k, const hla::Mat& H) {
    if (k == 0 || b == 0) return;
    double* hd = scratch(kSlotUpd, H.size());
    double* hp = pinned(H.size());
    STKG_CUDA_CHECK(cudaStreamSynchronize(s_));  // the pinned staging buffer is reused
    std::copy(H.begin(), H.end(), hp);
    STKG_CUDA_CHECK(cudaMemcpyAsync(hd, hp, sizeof(double) * H.size(), cudaMemcpyHostToDevice, s_));
    update_dev(W, b, V, k, hd);
  }

  // out (n x p) = W (n x q) * S (q x p, host column-major)
  void small_gemm(const double* W, int64_t q, const hla::Mat& S, int64_t p, double* out) {
    double* sdp = scratch(kSlotGemm, S.size());
    double* hp = pinned(S.size());
    STKG_CUDA_CHECK(cudaStreamSynchronize(s_));
    std::copy(S.begin(), S.end(), hp);
    STKG_CUDA_CHECK(cudaMemcpyAsync(sdp, hp, sizeof(double) * S.size(), cudaMemcpyHostToDevice, s_));
    GemmProblem g;
    g.M = n_;
    g.K = q;
    g.N = p;
    g.A = W;
    g.lda = n_;
    g.B = sdp;
    g.ldb = q;
    g.C = out;
    g.ldc = n_;
    launch_gemm(g, EpiStore{}, s_);
    STKG_CUDA_CHECK(cudaGetLastError());
  }

  void apply_M(const double* X, double* out, int64_t b) {  // out = M X (column-wise)
    for (int64_t j0 = 0; j0 < b; j0 += kTsRhs) {
      const int64_t bb = std::min<int64_t>(kTsRhs, b - j0);
      apply_with_time(h_, X + j0 * n_, out + j0 * n_, bb, ones_.p, zeros_.p, zeros_.p, zeros_.p);
    }
  }
  void apply_A(const double* X, double* out, int64_t b) {  // out = A X
    for (int64_t j0 = 0; j0 < b; j0 += kTsRhs) {
      const int64_t bb = std::min<int64_t>(kTsRhs, b - j0);
      apply_with_time(h_, X + j0 * n_, out + j0 * n_, bb, zeros_.p, zeros_.p, ones_.p, zeros_.p);
    }
  }

  // out = (A - sigma M)^-1 M X  (stk/rksm.hpp:211), X n x b
  void shifted_solve(const double* X, double* out, int64_t b, double sigma) {
    if (h_.ndim == 1) {  // batched tridiagonal solves
      apply_M(X, out, b);
      double* cp = scratch(kSlotT0, static_cast<size_t>(n_ * b));
      thomas_kernel<<<static_cast<unsigned>(ceil_div(b, 32)), 32, 0, s_>>>(
          h_.m_diag[0].p, h_.m_off[0].p, h_.a_diag[0].p, h_.a_off[0].p, n_, sigma, out,
          static_cast<int>(b), cp);
      STKG_CUDA_CHECK(cudaGetLastError());
      return;
    }
    // tensor eigenbasis: X (Lambda - sigma)^-1 X^T M  (dense)  /  S (Lambda - sigma)^-1 S (P1 DST)
    double* t0 = scratch(kSlotT0, static_cast<size_t>(n_ * b));
    double* t1 = scratch(kSlotT1, static_cast<size_t>(n_ * b));
    const bool dst = h_.transform == STKG_TRANSFORM_P1_DST;
    const double* src = X;
    if (!dst) {  // X^T M W needs M W; in the sine basis X^T M = diag(mu^1/2) S cancels
      apply_M(X, t1, b);
      src = t1;
    }
    for (int a = h_.ndim - 1; a >= 0; --a) {  // forward transforms
      double* dstp = (src == t0) ? t1 : t0;
      axis_pass(h_, a, true, src, dstp, b);
      src = dstp;
    }
    scale_modes_kernel<<<ew_blocks(), 256, 0, s_>>>(const_cast<double*>(src), n_, static_cast<int>(b),
                                            mode_lambda(h_), sigma);
    STKG_CUDA_CHECK(cudaGetLastError());
    for (int a = 0; a < h_.ndim; ++a) {  // inverse transforms
      double* dstp = (a == h_.ndim - 1) ? out : (src == t0 ? t1 : t0);
      axis_pass(h_, a, false, src, dstp, b);
      src = dstp;
    }
  }

  // Rank-revealing orthonormalisation of W (n x b) in place -- the role of
  // ColPivHouseholderQR with setThreshold(tol) (stk/rksm.hpp:146-151, :214-224): column-pivoted
  // Gram-Schmidt (largest remaining column first), every projection applied twice, and a
  // DGKS re-orthogonalisation of the accepted column against `prev` (k_prev columns) and the
  // columns already accepted when its norm dropped below half of its original.  A column is
  // accepted while its remaining norm exceeds tol * (largest original column norm), i.e.
  // while |R_ii| > tol |R_00|.  The accepted columns end up in W(:, 0:rank); Rout (rank x b,
  // original column order) = Q^T W_original.
  int orthonormalize(double* W, int64_t b, double tol, hla::Mat* Rout,
                     const double* prev = nullptr, int64_t k_prev = 0) {
    double* w0 = nullptr;
    if (Rout) {
      w0 = scratch(kSlotW0, static_cast<size_t>(n_ * b));
      STKG_CUDA_CHECK(cudaMemcpyAsync(w0, W, sizeof(double) * n_ * b, cudaMemcpyDeviceToDevice, s_));
    }
    std::vector<int> orig(b);  // original column index at each position
    for (int64_t j = 0; j < b; ++j) orig[j] = static_cast<int>(j);
    std::vector<double> norm0(b);
    double maxpiv = 0.0;
    hla::Mat G0 = gram(W, b, W, b);  // also the first step's Gram (saves a round trip)
    for (int64_t j = 0; j < b; ++j) {
      norm0[j] = std::sqrt(std::max(G0[j * b + j], 0.0));
      maxpiv = std::max(maxpiv, norm0[j]);
    }
    double* tmp = scratch(kSlotTmp, static_cast<size_t>(n_));
    int r = 0;
    while (r < b && maxpiv > 0.0) {
      const int64_t m = b - r;
      hla::Mat G = r == 0 ? G0 : gram(W + r * n_, m, W + r * n_, m);
      int64_t p = 0;
      for (int64_t j = 1; j < m; ++j)
        if (G[j * m + j] > G[p * m + p]) p = j;
      double nrm = std::sqrt(std::max(G[p * m + p], 0.0));
      if (!(nrm > tol * maxpiv)) break;
      if (p != 0) {  // move the pivot column to position r
        double* a = W + r * n_;
        double* c = W + (r + p) * n_;
        STKG_CUDA_CHECK(cudaMemcpyAsync(tmp, a, sizeof(double) * n_, cudaMemcpyDeviceToDevice, s_));
        STKG_CUDA_CHECK(cudaMemcpyAsync(a, c, sizeof(double) * n_, cudaMemcpyDeviceToDevice, s_));
        STKG_CUDA_CHECK(cudaMemcpyAsync(c, tmp, sizeof(double) * n_, cudaMemcpyDeviceToDevice, s_));
        std::swap(orig[r], orig[r + p]);
      }
      double* q = W + r * n_;
      if (nrm < 0.5 * norm0[orig[r]]) {  // DGKS: cancellation -> one more full projection
        // (coefficients stay on the device: no host round trip until the norm)
        if (k_prev > 0) project_out(q, 1, prev, k_prev);
        if (r > 0) project_out(q, 1, W, r);
        nrm = std::sqrt(std::max(gram(q, 1, q, 1)[0], 0.0));
        if (!(nrm > tol * maxpiv)) break;
      }
      scale(q, 1.0 / nrm);
      if (m > 1)
        for (int pass = 0; pass < 2; ++pass) project_out(q + n_, m - 1, q, 1);
      ++r;
    }
    if (Rout) {
      Rout->assign(static_cast<size_t>(std::max(r, 1)) * b, 0.0);
      if (r > 0) {
        hla::Mat Rt = gram(W, r, w0, b);  // r x b, original order
        std::copy(Rt.begin(), Rt.end(), Rout->begin());
      }
    }
    return r;
  }

  void scale(double* x, double alpha) {
    scale_kernel<<<ew_blocks(), 256, 0, s_>>>(x, n_, alpha);
    STKG_CUDA_CHECK(cudaGetLastError());
  }

  // W(:, 0:b) -= V(:, 0:k) (V^T W) with the coefficients kept on the device.
  void project_out(double* W, int64_t b, const double* V, int64_t k) {
    if (k == 0 || b == 0) return;
    double* hd = scratch(kSlotGs, static_cast<size_t>(k * b));
    gram_dev(V, k, W, b, hd);
    update_dev(W, b, V, k, hd);
  }

  // Two block classical Gram-Schmidt passes of W (n x b) against V(:, 0:k) (:213)
  void block_gs(double* W, int64_t b, const double* V, int64_t k) {
    if (k == 0) return;
    double* hd = scratch(kSlotGs, static_cast<size_t>(k * b));
    for (int pass = 0; pass < 2; ++pass) {
      gram_dev(V, k, W, b, hd);
      update_dev(W, b, V, k, hd);
    }
  }

  // --------------------------------------------------------------- the solver ------
  void run(int64_t rank, const double* L, const double* R, double* U_left, double* U_right,
           int64_t cap, int64_t* rank_out, stkg_report* rep);

 private:
  stkg_heat& h_;
  stkg_rksm_options o_;
  int64_t n_, nt_;
  cudaStream_t s_;
  // workspace lives in the plan (stkg_heat::rk_*) and persists across calls
  DevBuf &partials_, &hdev_, &ones_, &zeros_;
  enum { kSlotGram, kSlotUpd, kSlotGemm, kSlotT0, kSlotT1, kSlotW0, kSlotTmp, kSlotGs, kSlotRes,
         kSlots };
  static_assert(kSlots <= 16, "stkg_heat::rk_slots");
  DevBuf* slots_;
  double*& hpin_;
  size_t& hpin_n_;
};

// adaptive_next_shift (stk/rksm.hpp:67-102): 200 log-spaced candidates in
// [-2 lam_max, -lam_min/2], maximise the rational misfit, ties toward the smallest |x|.
double next_shift(const std::vector<double>& shifts, const std::vector<double>& ritz,
                  double lam_min, double lam_max) {
  const int nc = 200;
  const double lo = std::log(lam_min / 2.0), hi = std::log(2.0 * lam_max);
  double best = 0.0, best_val = -std::numeric_limits<double>::infinity();
  bool first = true;
  for (int i = 0; i < nc; ++i) {
    const double x = -std::exp(lo + (hi - lo) * i / (nc - 1));
    if (first) {
      best = x;
      first = false;
    }
    double val = 0.0;
    for (double s : shifts) {
      const double d = std::abs(x - s);
      if (d == 0.0) {
        val = -std::numeric_limits<double>::infinity();
        break;
      }
      val += std::log(d);
    }
    for (double lam : ritz) val -= std::log(std::max(std::abs(x + lam), 1e-300));
    if (val > best_val || (val == best_val && std::abs(x) < std::abs(best))) {
      best_val = val;
      best = x;
    }
  }
  return best;
}

// solve_projected_heat_with (stk/sylvester.hpp:117-142) for the small projected system:
// X (k x k), lambdas, G (k x nt) -> Y (k x nt)
hla::Mat projected_heat(const hla::Mat& X, const std::vector<double>& lam, const stkg_heat& h,
                        const hla::Mat& G, int k) {
  const int nt = static_cast<int>(h.nt);
  hla::Mat XT = hla::transpose(X, k, k);
  hla::Mat gt = hla::matmul(XT, G, k, k, nt);
  hla::Mat yt(static_cast<size_t>(k) * nt);
  for (int i = 0; i < k; ++i) {
    const double l = lam[i];
    for (int j = 0; j < nt; ++j) {
      const double piv = h.d_diag_h[j] + l * h.c_diag_h[j];
      if (std::abs(piv) < 1e-300)
        throw Error(STKG_SINGULARITY, "solve_projected_heat: singular row system at lambda = " +
                                          std::to_string(l));
      double rhs = gt[static_cast<size_t>(j) * k + i];
      if (j > 0) rhs -= (h.d_sup_h[j - 1] + l * h.c_sup_h[j - 1]) * yt[static_cast<size_t>(j - 1) * k + i];
      yt[static_cast<size_t>(j) * k + i] = rhs / piv;
    }
  }
  return hla::matmul(X, yt, k, k, nt);
}

// Optional per-phase wall-clock breakdown (STKG_RKSM_TIMING=1: synchronises at each mark
// and prints the totals to stderr at the end of the solve).
struct PhaseTimer {
  bool on = std::getenv("STKG_RKSM_TIMING") != nullptr;
  cudaStream_t s = nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  void mark(int phase) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto t = std::chrono::steady_clock::now();
    acc[phase] += std::chrono::duration<double>(t - t0).count();
    t0 = t;
  }
  void print() const {
    if (!on) return;
    static const char* names[8] = {"apply M,A", "projections", "residual basis", "T update",
                                   "pencil+projected", "residual norm", "shifted solve",
                                   "expansion GS+QR"};
    for (int i = 0; i < 8; ++i) std::fprintf(stderr, "rksm %-18s %8.3f s\n", names[i], acc[i]);
  }
};

void report_push(stkg_report* rep, double v) {
  if (!rep) return;
  if (rep->rel_res_history && rep->history_length < rep->history_capacity)
    rep->rel_res_history[rep->history_length] = v;
  rep->history_length++;
}

void Rksm::run(int64_t rank, const double* L, const double* R, double* U_left, double* U_right,
               int64_t cap, int64_t* rank_out, stkg_report* rep) {
  const auto t_start = std::chrono::steady_clock::now();
  const int nt = static_cast<int>(nt_);
  if (rep) {
    rep->iterations = 0;
    rep->mu_mem = 0;
    rep->converged = 0;
    rep->stagnated = 0;
    rep->final_relres = 0.0;
    rep->history_length = 0;
  }
  // right factor of F on the host (n_t x rank)
  hla::Mat Rh(static_cast<size_t>(nt_ * rank));
  STKG_CUDA_CHECK(cudaMemcpyAsync(Rh.data(), R, sizeof(double) * Rh.size(), cudaMemcpyDeviceToHost, s_));
  // full-column-rank left factor (:146-151): F = f1 f2^T with f1 orthonormal
  Block V;
  V.n = n_;
  V.reserve(std::max<int64_t>(rank * 4, 16), s_);
  STKG_CUDA_CHECK(cudaMemcpyAsync(V.col(0), L, sizeof(double) * n_ * rank, cudaMemcpyDeviceToDevice, s_));
  hla::Mat Rl;
  const int rf = orthonormalize(V.col(0), rank, 1e-13, &Rl);
  // f2 = R * Rl^T  (n_t x rf); ||F|| = ||f2|| since f1 has orthonormal columns
  hla::Mat RlT = hla::transpose(Rl, std::max(rf, 1), static_cast<int>(rank));
  hla::Mat f2 = rf > 0 ? hla::matmul(Rh, RlT, nt, static_cast<int>(rank), rf) : hla::Mat();
  const double norm_f = rf > 0 ? hla::frob(f2) : 0.0;
  if (norm_f == 0.0) {
    *rank_out = 0;
    if (rep) rep->converged = 1;
    return;
  }
  V.cols = rf;
  // exact spectral interval of the tensor pencil, widened like estimate_spectral_interval
  double lmin = 0.0, lmax = 0.0;
  for (int a = 0; a < h_.ndim; ++a) {
    lmin += *std::min_element(h_.lam_h[a].begin(), h_.lam_h[a].end());
    lmax += *std::max_element(h_.lam_h[a].begin(), h_.lam_h[a].end());
  }
  const double lam_min = lmin / 2.0, lam_max = 2.0 * lmax;

  Block MV, AV, Q;  // M V, A V and the orthonormal basis of span[f1, MV, AV]
  MV.n = AV.n = Q.n = n_;
  Q.reserve(3 * rf + 16, s_);
  STKG_CUDA_CHECK(cudaMemcpyAsync(Q.col(0), V.col(0), sizeof(double) * n_ * rf, cudaMemcpyDeviceToDevice, s_));
  Q.cols = rf;
  // host state
  hla::Mat T0 = gram(Q.col(0), rf, V.col(0), rf);  // Q^T f1 (= I up to rounding)
  hla::Mat hm, ha;        // k x k projections (leading dimension kcap_h)
  hla::Mat vtf1;          // k x rf
  hla::Mat T = T0;        // (q x m) with m = rf + 2k columns [f1 | MV | AV]
  std::vector<double> shifts, ritz;
  int64_t k_done = 0;     // columns of V already projected
  int64_t newest0 = 0, newest_b = rf;
  hla::Mat y;             // k x nt
  int64_t kfinal = 0;
  bool converged = false;
  std::vector<double> history;
  const int total_iters = o_.fixed_iters > 0 ? o_.fixed_iters : o_.maxit;
  int it = 0;
  PhaseTimer tm;
  tm.s = s_;
  for (it = 1; it <= total_iters; ++it) {
    const int64_t k = V.cols, b = k - k_done;
    tm.mark(7);
    // --- M V_new, A V_new
    MV.reserve(k, s_);
    AV.reserve(k, s_);
    apply_M(V.col(k_done), MV.col(k_done), b);
    apply_A(V.col(k_done), AV.col(k_done), b);
    MV.cols = AV.cols = k;
    tm.mark(0);
    // --- projections V^T M V, V^T A V grown by the new columns (:180-183)
    {
      // one device->host read for V^T M V_new, V^T A V_new and V_new^T f1
      auto g3 = gram_batch({{V.col(0), k, MV.col(k_done), b},
                            {V.col(0), k, AV.col(k_done), b},
                            {V.col(k_done), b, V.col(0), rf}});
      hla::Mat& cm = g3[0];  // k x b
      hla::Mat& ca = g3[1];
      hla::Mat nhm(static_cast<size_t>(k * k)), nha(static_cast<size_t>(k * k));
      for (int64_t j = 0; j < k_done; ++j)
        for (int64_t i = 0; i < k_done; ++i) {
          nhm[j * k + i] = hm[j * k_done + i];
          nha[j * k + i] = ha[j * k_done + i];
        }
      for (int64_t j = 0; j < b; ++j)
        for (int64_t i = 0; i < k; ++i) {
          const double vm = cm[j * k + i], va = ca[j * k + i];
          nhm[(k_done + j) * k + i] = vm;
          nha[(k_done + j) * k + i] = va;
          if (i < k_done) {  // mirror into the new rows
            nhm[i * k + k_done + j] = vm;
            nha[i * k + k_done + j] = va;
          }
        }
      // symmetrise the new diagonal block (:182-183)
      for (int64_t j = 0; j < b; ++j)
        for (int64_t i = 0; i < j; ++i) {
          const int64_t r = k_done + i, c = k_done + j;
          const double sm = 0.5 * (nhm[c * k + r] + nhm[r * k + c]);
          const double sa = 0.5 * (nha[c * k + r] + nha[r * k + c]);
          nhm[c * k + r] = nhm[r * k + c] = sm;
          nha[c * k + r] = nha[r * k + c] = sa;
        }
      hm.swap(nhm);
      ha.swap(nha);
      // V_new^T f1
      hla::Mat nf(static_cast<size_t>(k * rf));
      for (int64_t j = 0; j < rf; ++j)
        for (int64_t i = 0; i < k_done; ++i) nf[j * k + i] = vtf1[j * k_done + i];
      hla::Mat& cf = g3[2];  // b x rf
      for (int64_t j = 0; j < rf; ++j)
        for (int64_t i = 0; i < b; ++i) nf[j * k + k_done + i] = cf[j * b + i];
      vtf1.swap(nf);
    }
    tm.mark(1);
    // --- residual basis: orthonormalise [MV_new, AV_new] against Q and append
    const int64_t q_old = Q.cols;
    {
      double* wres = scratch(kSlotRes, static_cast<size_t>(n_ * 2 * b));
      STKG_CUDA_CHECK(cudaMemcpyAsync(wres, MV.col(k_done), sizeof(double) * n_ * b, cudaMemcpyDeviceToDevice, s_));
      STKG_CUDA_CHECK(cudaMemcpyAsync(wres + n_ * b, AV.col(k_done), sizeof(double) * n_ * b, cudaMemcpyDeviceToDevice, s_));
      block_gs(wres, 2 * b, Q.col(0), Q.cols);
      const int add = orthonormalize(wres, 2 * b, 1e-12, nullptr, Q.col(0), Q.cols);
      if (add > 0) {
        Q.reserve(Q.cols + add, s_);
        STKG_CUDA_CHECK(cudaMemcpyAsync(Q.col(Q.cols), wres, sizeof(double) * n_ * add, cudaMemcpyDeviceToDevice, s_));
        Q.cols += add;
      }
    }
    tm.mark(2);
    // --- T = Q^T [f1 | MV | AV]: (q x m), grown by new rows and new columns
    {
      const int64_t q = Q.cols, m = rf + 2 * k, m_old = rf + 2 * k_done;
      hla::Mat nT(static_cast<size_t>(q * m), 0.0);
      // old block: rows < q_old, columns f1 (rf), MV(0:k_done), AV(0:k_done)
      for (int64_t j = 0; j < m_old; ++j) {
        const int64_t jn = j < rf ? j : (j < rf + k_done ? j : j + b);  // AV shifts by b
        for (int64_t i = 0; i < q_old; ++i) nT[jn * q + i] = T[j * q_old + i];
      }
      // new rows for old columns: Q_new^T [f1 | MV_old | AV_old]
      const int64_t qn = q - q_old;
      if (qn > 0) {
        auto ga = gram_batch({{Q.col(q_old), qn, V.col(0), rf},
                              {Q.col(q_old), qn, MV.col(0), k_done},
                              {Q.col(q_old), qn, AV.col(0), k_done}});
        hla::Mat& a1 = ga[0];
        hla::Mat& a2 = ga[1];
        hla::Mat& a3 = ga[2];
        for (int64_t j = 0; j < rf; ++j)
          for (int64_t i = 0; i < qn; ++i) nT[j * q + q_old + i] = a1[j * qn + i];
        for (int64_t j = 0; j < k_done; ++j)
          for (int64_t i = 0; i < qn; ++i) {
            nT[(rf + j) * q + q_old + i] = a2[j * qn + i];
            nT[(rf + k + j) * q + q_old + i] = a3[j * qn + i];
          }
      }
      // new columns (all rows): Q^T MV_new, Q^T AV_new
      auto gb = gram_batch({{Q.col(0), q, MV.col(k_done), b}, {Q.col(0), q, AV.col(k_done), b}});
      hla::Mat& b2 = gb[0];
      hla::Mat& b3 = gb[1];
      for (int64_t j = 0; j < b; ++j)
        for (int64_t i = 0; i < q; ++i) {
          nT[(rf + k_done + j) * q + i] = b2[j * q + i];
          nT[(rf + k + k_done + j) * q + i] = b3[j * q + i];
        }
      T.swap(nT);
    }
    k_done = k;
    tm.mark(3);
    // --- projected pencil and projected heat solve (:184-188)
    hla::Mat X(static_cast<size_t>(k * k));
    std::vector<double> lam(k);
    {
      const int st = stkg_sym_gen_eig(static_cast<int>(k), ha.data(), hm.data(), lam.data(), X.data());
      if (st != STKG_OK) throw Error(st, stkg_last_error_message());
    }
    ritz = lam;
    hla::Mat f2T = hla::transpose(f2, nt, rf);
    hla::Mat g = hla::matmul(vtf1, f2T, static_cast<int>(k), rf, nt);  // k x nt
    y = projected_heat(X, lam, h_, g, static_cast<int>(k));
    kfinal = k;
    tm.mark(4);
    // --- factored residual (:190-191): ||T W^T|| with W = [f2 | -D^T y^T | -C^T y^T]
    {
      const int64_t q = Q.cols, m = rf + 2 * k;
      hla::Mat W(static_cast<size_t>(nt * m));
      for (int64_t j = 0; j < rf; ++j)
        for (int t = 0; t < nt; ++t) W[j * nt + t] = f2[j * nt + t];
      for (int64_t c = 0; c < k; ++c)
        for (int t = 0; t < nt; ++t) {
          // (D^T y^T)[t, c] = sum_s D[s, t] y[c, s] = d_diag[t] y[c,t] + d_sup[t-1] y[c,t-1]
          const double yc = y[static_cast<size_t>(t) * k + c];
          const double yp = t > 0 ? y[static_cast<size_t>(t - 1) * k + c] : 0.0;
          const double dv = h_.d_diag_h[t] * yc + (t > 0 ? h_.d_sup_h[t - 1] * yp : 0.0);
          const double cv = h_.c_diag_h[t] * yc + (t > 0 ? h_.c_sup_h[t - 1] * yp : 0.0);
          W[(rf + c) * nt + t] = -dv;
          W[(rf + k + c) * nt + t] = -cv;
        }
      hla::Mat WT = hla::transpose(W, nt, static_cast<int>(m));
      hla::Mat Rres = hla::matmul(T, WT, static_cast<int>(q), static_cast<int>(m), nt);
      const double relres = hla::frob(Rres) / norm_f;
      history.push_back(relres);
      report_push(rep, relres);
      if (rep) rep->mu_mem = std::max<int>(rep->mu_mem, static_cast<int>(k + rf));
      if (o_.fixed_iters <= 0 && relres <= o_.tol) {
        converged = true;
        break;
      }
      if (it == total_iters) {
        converged = o_.fixed_iters > 0 || relres <= o_.tol;
        break;
      }
    }
    tm.mark(5);
    // --- next pole and space expansion (:193-224)
    const double sigma = shifts.empty() ? -lam_max : next_shift(shifts, ritz, lam_min, lam_max);
    shifts.push_back(sigma);
    V.reserve(k + newest_b, s_);
    double* w = V.col(k);
    shifted_solve(V.col(newest0), w, newest_b, sigma);
    tm.mark(6);
    block_gs(w, newest_b, V.col(0), k);
    const int add = orthonormalize(w, newest_b, 1e-12, nullptr, V.col(0), k);
    if (add == 0) {
      converged = o_.fixed_iters <= 0 && history.back() <= o_.tol;
      break;  // space exhausted
    }
    newest0 = k;
    newest_b = add;
    V.cols = k + add;
  }
  tm.mark(7);
  tm.print();
  if (rep) rep->iterations = std::min(it, total_iters);
  if (const char* dir = std::getenv("STKG_RKSM_DUMP")) {  // debugging aid: raw basis dump
    auto dump = [&](const char* name, const double* d, int64_t count, bool device) {
      std::vector<double> hbuf(static_cast<size_t>(count));
      if (device) {
        STKG_CUDA_CHECK(cudaMemcpy(hbuf.data(), d, sizeof(double) * count, cudaMemcpyDeviceToHost));
      } else {
        std::copy(d, d + count, hbuf.begin());
      }
      const std::string path = std::string(dir) + "/" + name + ".bin";
      if (FILE* f = std::fopen(path.c_str(), "wb")) {
        std::fwrite(hbuf.data(), sizeof(double), hbuf.size(), f);
        std::fclose(f);
      }
    };
    dump("V", V.col(0), V.cols * n_, true);
    dump("MV", MV.col(0), MV.cols * n_, true);
    dump("AV", AV.col(0), AV.cols * n_, true);
    dump("Q", Q.col(0), Q.cols * n_, true);
    dump("T", T.data(), static_cast<int64_t>(T.size()), false);
    dump("y", y.data(), static_cast<int64_t>(y.size()), false);
    std::vector<double> dims = {double(n_), double(V.cols), double(MV.cols), double(Q.cols), double(kfinal), double(rf)};
    dump("dims", dims.data(), 6, false);
  }
  // --- lowrank_truncate(V, y^T, final_tol) (:226-228): V orthonormal, so the SVD of y
  const double final_tol = o_.fixed_iters > 0 ? o_.trunc_tol : o_.tol;
  const int k = static_cast<int>(kfinal);
  hla::Mat yT = hla::transpose(y, k, nt);  // nt x k
  std::vector<double> sv;
  hla::Mat Uy, Vy;  // y^T = Uy diag(sv) Vy^T  =>  U = V y = V Vy diag(sv) Uy^T
  if (nt >= k) {
    hla::jacobi_svd(yT, nt, k, sv, Uy, Vy);
  } else {
    hla::jacobi_svd(y, k, nt, sv, Vy, Uy);  // y = Vy diag Uy^T
  }
  const int r = static_cast<int>(sv.size());
  double total2 = 0.0;
  for (double s2 : sv) total2 += s2 * s2;
  int keep = r;
  if (total2 == 0.0) {
    keep = 0;
  } else {
    const double budget2 = final_tol * final_tol * total2;
    double tail2 = 0.0;
    while (keep > 0) {
      const double next = tail2 + sv[keep - 1] * sv[keep - 1];
      if (next > budget2) break;
      tail2 = next;
      --keep;
    }
  }
  *rank_out = keep;
  STKG_REQUIRE(keep <= cap, STKG_ARGUMENT, "rksm: solution rank exceeds the output capacity");
  if (keep > 0) {
    // left = V Vy(:, :keep) diag(sv) ; right = Uy(:, :keep)   (k x keep and nt x keep)
    hla::Mat Z(static_cast<size_t>(k) * keep);
    for (int c = 0; c < keep; ++c)
      for (int i = 0; i < k; ++i) Z[static_cast<size_t>(c) * k + i] = Vy[static_cast<size_t>(c) * k + i] * sv[c];
    small_gemm(V.col(0), k, Z, keep, U_left);
    STKG_CUDA_CHECK(cudaMemcpyAsync(U_right, Uy.data(), sizeof(double) * nt * keep, cudaMemcpyHostToDevice, s_));
    STKG_CUDA_CHECK(cudaStreamSynchronize(s_));
  }
  if (rep) {
    rep->converged = converged ? 1 : 0;
    rep->final_relres = history.empty() ? 0.0 : history.back();
    rep->wall_time_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  }
}

}  // namespace

extern "C" int stkg_heat_rksm(stkg_heat* plan, int64_t rank, const double* L, const double* R,
                              const stkg_rksm_options* opts, double* U_left, double* U_right,
                              int64_t cap, int64_t* rank_out, stkg_report* report) {
  return guarded([&] {
    STKG_REQUIRE(plan && L && R && U_left && U_right && rank_out, STKG_ARGUMENT,
                 "rksm_solve: null argument");
    STKG_REQUIRE(rank >= 1, STKG_ARGUMENT, "rksm_solve: F shape mismatch");
    STKG_REQUIRE(plan->has_operator, STKG_ARGUMENT,
                 "rksm_solve: plan was created without the spatial factors");
    stkg_rksm_options o = opts ? *opts : stkg_rksm_options{1e-8, 100, 0, 1e-10};
    STKG_REQUIRE(o.fixed_iters >= 0, STKG_ARGUMENT, "rksm_solve: fixed_iters must be >= 1");
    STKG_REQUIRE(o.maxit >= 1, STKG_ARGUMENT, "rksm_solve: maxit must be >= 1");
    // lowrank_truncate's argument check (stk/la_core.hpp:135) on the tolerance the final
    // truncation uses (stk/rksm.hpp:226-227), made before any work is done
    const double final_tol = o.fixed_iters > 0 ? o.trunc_tol : o.tol;
    STKG_REQUIRE(final_tol > 0.0 && final_tol < 1.0, STKG_ARGUMENT,
                 "lowrank_truncate: tol must be in (0,1)");
    Rksm solver(*plan, o);
    solver.run(rank, L, R, U_left, U_right, cap, rank_out, report);
  });
}
