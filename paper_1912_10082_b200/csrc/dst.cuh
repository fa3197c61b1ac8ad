// Fast sine transform backend for the uniform-P1 eigenbasis.
//
// For P1 elements on a uniform grid with n interior nodes (N = n + 1), the generalized
// eigenbasis of (A_h, M_h) is X = S diag(mu^-1/2) with S[i,k] = sqrt(2/N) sin(pi i k / N)
// the orthonormal DST-I matrix (S = S^T = S^-1) and mu_k = (h/3)(2 + cos(pi k / N)) the
// eigenvalues of M_h.  The dense transforms X^T F and X Y of solve_projected_heat_with
// (stk/sylvester.hpp:126,141) are therefore a DST-I along each axis plus a diagonal
// scaling; the scaling mu^-1 (both directions) is folded into the modal recurrence.
//
// DST-I of two real vectors a, b (length N-1) at once: with c_j = a_j + i b_j (j = 1..N-1,
// zero elsewhere) and W = FFT_{2N}(c),
//     DST(a)_k = -(Im W_k - Im W_{2N-k}) / 2,   DST(b)_k = (Re W_k - Re W_{2N-k}) / 2.
// The length-2N complex FFT runs in shared memory as a Stockham auto-sort FFT with radix-8
// stages (radix-4/2 last), twiddles from a table of 2N-th roots of unity built on the host
// with exact integer argument reduction.  Cost: 5 (2N) log2(2N) flop per pair, i.e. about
// 5 log2(2N) flop per element -- O(log n) instead of the 2n of a dense transform.
#pragma once

#include "common.cuh"
#include "gemm_f64.cuh"  // cp_async8 / commit / wait


namespace stkg {

// Complex helpers (double2 = (re, im))
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 mul_neg_i(double2 a) { return make_double2(a.y, -a.x); }  // -i a

// Forward DFT of size 4: Y_q = sum_r c_r exp(-2 pi i r q / 4)
__device__ __forceinline__ void dft4(double2& c0, double2& c1, double2& c2, double2& c3) {
  const double2 s02 = cadd(c0, c2), d02 = csub(c0, c2);
  const double2 s13 = cadd(c1, c3), d13 = mul_neg_i(csub(c1, c3));
  c0 = cadd(s02, s13);
  c2 = csub(s02, s13);
  c1 = cadd(d02, d13);
  c3 = csub(d02, d13);
}

// Forward DFT of size 8 (decimation in frequency into two size-4 DFTs); output in
// natural order in v[0..7].
__device__ __forceinline__ void dft8(double2 (&v)[8]) {
  constexpr double r2 = 0.70710678118654752440;  // 1/sqrt(2)
  double2 a[4], b[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    a[r] = cadd(v[r], v[r + 4]);
    b[r] = csub(v[r], v[r + 4]);
  }
  // b_r *= w^r, w = exp(-2 pi i / 8)
  b[1] = make_double2((b[1].x + b[1].y) * r2, (b[1].y - b[1].x) * r2);
  b[2] = mul_neg_i(b[2]);
  b[3] = make_double2((b[3].y - b[3].x) * r2, -(b[3].x + b[3].y) * r2);
  dft4(a[0], a[1], a[2], a[3]);
  dft4(b[0], b[1], b[2], b[3]);
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    v[2 * p] = a[p];
    v[2 * p + 1] = b[p];
  }
}

template <int R>
__device__ __forceinline__ void dft_radix(double2 (&v)[R]);
template <>
__device__ __forceinline__ void dft_radix<8>(double2 (&v)[8]) { dft8(v); }
template <>
__device__ __forceinline__ void dft_radix<4>(double2 (&v)[4]) { dft4(v[0], v[1], v[2], v[3]); }
template <>
__device__ __forceinline__ void dft_radix<2>(double2 (&v)[2]) {
  const double2 t = v[0];
  v[0] = cadd(t, v[1]);
  v[1] = csub(t, v[1]);
}

constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }

// Shared-memory index with one pad slot per 8 complex values: the stride-8 (and stride-Ns)
// Stockham writes then spread over all banks instead of hitting one 128-byte bank group.
__host__ __device__ constexpr int pidx(int i) { return i + (i >> 3); }
template <int L>
constexpr int padded_len() { return L + L / 8; }

// One Stockham stage of radix R over NFFT FFTs of length L stored back to back in buf.
// NS = product of the radices of the previous stages, a compile-time constant so that the
// padded shared-memory index arithmetic folds into constant offsets.  In place: every
// thread reads its inputs, the block synchronises, then the outputs are written.
template <int L, int NFFT, int R, int THREADS, int NS>
__device__ __forceinline__ void stockham_stage(double2* buf, const double2* __restrict__ tw) {
  constexpr int kBut = L / R;                 // butterflies per FFT
  constexpr int total = NFFT * kBut;
  constexpr int kMaxPer = (total + THREADS - 1) / THREADS;
  constexpr int stride = L / (NS * R);        // twiddle index step
  double2 v[kMaxPer][R];
#pragma unroll
  for (int u = 0; u < kMaxPer; ++u) {
    const int t = threadIdx.x + u * THREADS;
    if (total % THREADS == 0 || t < total) {
      const int f = t / kBut, j = t % kBut;
      const double2* x = buf + f * padded_len<L>();
      const int k = j % NS;
      // one table load per butterfly: w = exp(-2 pi i k / (NS R)); w^r by multiplication
      // (a few ulps, far below the 1e-10 parity bar) instead of R-1 L1 loads
      double2 wr = make_double2(1.0, 0.0);
      const double2 w = (NS > 1 && k > 0) ? __ldg(tw + k * stride) : make_double2(1.0, 0.0);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double2 val = x[pidx(j + r * kBut)];
        if (NS > 1 && r > 0) {
          wr = r == 1 ? w : cmul(wr, w);
          if (k > 0) val = cmul(val, wr);
        }
        v[u][r] = val;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kMaxPer; ++u) {
    const int t = threadIdx.x + u * THREADS;
    if (total % THREADS == 0 || t < total) {
      const int f = t / kBut, j = t % kBut;
      dft_radix<R>(v[u]);
      double2* y = buf + f * padded_len<L>();
      const int base = (j / NS) * NS * R + j % NS;
#pragma unroll
      for (int r = 0; r < R; ++r) y[pidx(base + r * NS)] = v[u][r];
    }
  }
  __syncthreads();
}

// Radix of the last stage of the length-L plan: floor(log8 L) radix-8 stages, then a
// radix-4 or -2 stage when log2 L is not a multiple of 3.
template <int L>
constexpr int last_radix() {
  return (L >> (3 * (ilog2(L) / 3))) == 1 ? 8 : (L >> (3 * (ilog2(L) / 3)));
}

// COUNT radix-8 stages starting at NS (compile-time recursion).
template <int L, int NFFT, int THREADS, int NS, int COUNT>
__device__ __forceinline__ void radix8_stages(double2* buf, const double2* tw) {
  if constexpr (COUNT > 0) {
    stockham_stage<L, NFFT, 8, THREADS, NS>(buf, tw);
    radix8_stages<L, NFFT, THREADS, NS * 8, COUNT - 1>(buf, tw);
  }
}

// The stages after the fused first radix-8 stage, excluding the last one (which is fused
// with the DST post-processing when it has radix 4).
template <int L, int THREADS>
__device__ __forceinline__ void fft_middle_stages(double2* buf, const double2* tw) {
  constexpr int kStages8 = ilog2(L) / 3;
  constexpr int kLast8 = last_radix<L>() == 8 ? 1 : 0;
  radix8_stages<L, 1, THREADS, 8, kStages8 - 1 - kLast8>(buf, tw);
}

// All stages after the fused first radix-8 stage.
template <int L, int NFFT, int THREADS>
__device__ __forceinline__ void fft_after_first_stage(double2* buf, const double2* tw) {
  constexpr int kStages8 = ilog2(L) / 3;
  constexpr int kTail = L >> (3 * kStages8);
  constexpr int kNsTail = 1 << (3 * kStages8);
  radix8_stages<L, NFFT, THREADS, 8, kStages8 - 1>(buf, tw);
  if constexpr (kTail == 2) stockham_stage<L, NFFT, 2, THREADS, kNsTail>(buf, tw);
  if constexpr (kTail == 4) stockham_stage<L, NFFT, 4, THREADS, kNsTail>(buf, tw);
}

// Last Stockham stage of radix 4 (Ns = L/4 butterflies, THREADS = L/8: two per thread)
// fused with the DST-I post-processing.  Thread t takes butterflies j1 = t and
// j2 = Ns - t (t = 0: j2 = Ns/2); the output pairs (W_k, W_{L-k}) then live in its own
// registers: k = j1 + r Ns pairs with L - k = j2 + (3 - r) Ns.  Writes ya_k, yb_k
// (k = 1..n) through `emit(k, ya, yb)`.
template <int L, int THREADS, class Emit>
__device__ __forceinline__ void last_radix4_stage_with_post(const double2* buf,
                                                            const double2* __restrict__ tw,
                                                            double hs, int n, Emit emit) {
  constexpr int Ns = L / 4;
  static_assert(THREADS * 2 == Ns, "two radix-4 butterflies per thread");
  const int t = threadIdx.x;
  const int jj[2] = {t, t == 0 ? Ns / 2 : Ns - t};
  double2 W[2][4];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int j = jj[u], k = j;  // j % Ns == j
    const double2 w = k > 0 ? __ldg(tw + k) : make_double2(1.0, 0.0);  // stride L/(Ns R) = 1
    double2 wr = w;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double2 val = buf[pidx(j + r * Ns)];
      if (r > 0) {
        if (r > 1) wr = cmul(wr, w);
        if (k > 0) val = cmul(val, wr);
      }
      W[u][r] = val;
    }
    dft4(W[u][0], W[u][1], W[u][2], W[u][3]);  // outputs j + r Ns, r = 0..3
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int k = jj[u] + r * Ns;
      if (k < 1 || k > n) continue;
      // partner W_{L-k}: (t >= 1) other butterfly, index 3 - r; (t == 0) same butterfly
      double2 pm;
      if (t > 0) pm = W[1 - u][3 - r];
      else pm = u == 0 ? W[0][(4 - r) & 3] : W[1][3 - r];
      emit(k, -hs * (W[u][r].y - pm.y), hs * (W[u][r].x - pm.x));
    }
  }
}

// Orthonormal DST-I along one axis of data viewed as [outer][n][inner] (element j of
// vector (o, i) at (o * n + j) * inner + i); vectors = outer * inner.  `scale` multiplies
// the result (sqrt(2/N)).  dst may alias src (a work item is read completely before any of
// it is written, and items are disjoint).
//
// Persistent CTAs walk over work items of two neighbouring vectors (one complex FFT).  The
// first FFT stage needs, per thread, the 4 nonzero inputs m = j + r L/8 (r < 4) of both
// vectors: those 8 doubles of the NEXT item are loaded into registers while the current
// item is transformed, so HBM latency hides behind the FFT without staging buffers.
template <int L>
struct DstLaunch {
  static constexpr int kThreads = L / 8;  // one radix-8 butterfly per thread per stage
  static constexpr int kCtasPerSm = 2048 / kThreads < 8 ? 2048 / kThreads : 8;
  static constexpr size_t kSmem = size_t(padded_len<L>()) * sizeof(double2);
};

template <int L>
__global__ void __launch_bounds__(L / 8, (L >= 2048 ? 2 : 3)) dst_axis_kernel(const double* __restrict__ src,
                                                         double* dst, int64_t n, int64_t inner,
                                                         int64_t nvec,
                                                         const double2* __restrict__ tw,
                                                         double scale) {
  constexpr int kThreads = L / 8;
  constexpr double r2 = 0.70710678118654752440;
  extern __shared__ __align__(16) double2 cbuf[];
  const int nn = static_cast<int>(n);
  const int64_t nitems = (nvec + 1) / 2;
  const int j = threadIdx.x;

  // first-stage inputs of an item: a[r] = vector 0, b[r] = vector 1 at m = j + r L/8
  auto fetch = [&](int64_t item, double (&a)[4], double (&b)[4], int64_t& b0, int64_t& b1) {
    b0 = b1 = -1;
    if (item < nitems) {
      const int64_t g0 = 2 * item, g1 = g0 + 1;
      b0 = (g0 / inner) * n * inner + g0 % inner;
      if (g1 < nvec) b1 = (g1 / inner) * n * inner + g1 % inner;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int m = j + r * kThreads;  // < L/2 = n + 1
      const bool in = m >= 1;
      const int64_t off = int64_t(m - 1) * inner;
      a[r] = (in && b0 >= 0) ? __ldcs(src + b0 + off) : 0.0;
      b[r] = (in && b1 >= 0) ? __ldcs(src + b1 + off) : 0.0;
    }
  };

  double na[4], nb[4];
  int64_t nb0, nb1;
  int64_t item = blockIdx.x;
  fetch(item, na, nb, nb0, nb1);
  const double hs = 0.5 * scale;
  for (; item < nitems; item += gridDim.x) {
    double2 v[4], w[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) v[r] = make_double2(na[r], nb[r]);
    const int64_t b0 = nb0, b1 = nb1;
    fetch(item + gridDim.x, na, nb, nb0, nb1);  // next item's loads in flight
    // stage 1 (Ns = 1): DFT-8 of (v0..v3, 0, 0, 0, 0)
#pragma unroll
    for (int r = 0; r < 4; ++r) w[r] = v[r];
    w[1] = make_double2((w[1].x + w[1].y) * r2, (w[1].y - w[1].x) * r2);
    w[2] = mul_neg_i(w[2]);
    w[3] = make_double2((w[3].y - w[3].x) * r2, -(w[3].x + w[3].y) * r2);
    dft4(v[0], v[1], v[2], v[3]);
    dft4(w[0], w[1], w[2], w[3]);
    __syncthreads();  // previous item's post-processing reads of cbuf are done
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      cbuf[pidx(j * 8 + 2 * q)] = v[q];
      cbuf[pidx(j * 8 + 2 * q + 1)] = w[q];
    }
    __syncthreads();
    if constexpr (last_radix<L>() == 4) {
      // middle stages, then the last radix-4 stage fused with the post-processing
      fft_middle_stages<L, kThreads>(cbuf, tw);
      last_radix4_stage_with_post<L, kThreads>(cbuf, tw, hs, nn, [&](int k, double ya, double yb) {
        if (b0 >= 0) __stcs(dst + b0 + int64_t(k - 1) * inner, ya);
        if (b1 >= 0) __stcs(dst + b1 + int64_t(k - 1) * inner, yb);
      });
    } else {
      fft_after_first_stage<L, 1, kThreads>(cbuf, tw);
      // post-process and store: both outputs k = e + 1 come from W_k and W_{L-k}
      for (int e = j; e < nn; e += kThreads) {
        const int k = e + 1;
        const double2 wk = cbuf[pidx(k)], wm = cbuf[pidx(L - k)];
        if (b0 >= 0) __stcs(dst + b0 + int64_t(e) * inner, -hs * (wk.y - wm.y));
        if (b1 >= 0) __stcs(dst + b1 + int64_t(e) * inner, hs * (wk.x - wm.x));
      }
    }
  }
}

// Strided axis (inner > 1): element j of vector (o, i) at (o * n + j) * inner + i.  A work
// item is a tile of G = 8 neighbouring vectors, so every row of the tile is 64 contiguous
// bytes (full DRAM bursts instead of 16-byte pieces).  Tiles are staged by cp.async into
// a double-buffered [G][n] shared-memory buffer (the next tile loads while this one is
// transformed), the G/2 complex FFTs read their inputs from and write their outputs back
// into the tile rows, and the tile leaves with coalesced 64-byte row stores.
template <int L>
struct DstStridedLaunch {
  static constexpr int kG = 8;
  static constexpr int kThreads = L / 8;
  static constexpr int kRow = L / 2;  // staging row pitch (>= n)
  // One staging buffer and 2 CTAs per SM: while one CTA waits for its tile the other one
  // transforms (a second buffer per CTA would halve the CTAs per SM).
  static constexpr int kBufs = 1;
  static constexpr size_t kSmem =
      size_t(padded_len<L>()) * sizeof(double2) + size_t(kBufs) * kG * kRow * sizeof(double);
};

template <int L>
__global__ void __launch_bounds__(L / 8, 2) dst_strided_kernel(
    const double* __restrict__ src, double* __restrict__ dst, int64_t n, int64_t inner,
    int64_t nvec, const double2* __restrict__ tw, double scale) {
  using C = DstStridedLaunch<L>;
  constexpr int G = C::kG, kThreads = C::kThreads, RP = C::kRow;
  constexpr double r2 = 0.70710678118654752440;
  extern __shared__ __align__(16) double2 cbuf[];
  double* stage = reinterpret_cast<double*>(cbuf + padded_len<L>());  // [2][G][RP]
  __shared__ int64_t vbase[2][G];
  const int nn = static_cast<int>(n);
  const int64_t ntiles = (nvec + G - 1) / G;
  const int j = threadIdx.x;

  auto tile_bases = [&](int buf, int64_t tile) {
    for (int v = threadIdx.x; v < G; v += kThreads) {  // kThreads may be < G (small L)
      const int64_t g = tile * G + v;
      vbase[buf][v] = (tile < ntiles && g < nvec) ? (g / inner) * n * inner + g % inner : -1;
    }
  };
  auto load_tile = [&](int buf) {  // rows of G consecutive doubles -> stage[buf][v][j]
    double* st = stage + buf * G * RP;
    for (int e = threadIdx.x; e < G * nn; e += kThreads) {
      const int v = e % G, jj = e / G;
      const int64_t b = vbase[buf][v];
      cp_async8(st + v * RP + jj, b >= 0 ? src + b + int64_t(jj) * inner : src, b >= 0);
    }
  };

  const double hs = 0.5 * scale;
  const int cur = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    __syncthreads();  // previous tile stored: vbase / stage are free
    tile_bases(0, tile);
    __syncthreads();
    load_tile(0);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();  // this tile has landed
    double* st = stage + cur * G * RP;
#pragma unroll 1
    for (int f = 0; f < G / 2; ++f) {
      double* ra = st + (2 * f) * RP;
      double* rb = st + (2 * f + 1) * RP;
      double2 v[4], w[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int m = j + r * kThreads;  // < L/2 = n + 1
        v[r] = (m >= 1) ? make_double2(ra[m - 1], rb[m - 1]) : make_double2(0.0, 0.0);
        w[r] = v[r];
      }
      w[1] = make_double2((w[1].x + w[1].y) * r2, (w[1].y - w[1].x) * r2);
      w[2] = mul_neg_i(w[2]);
      w[3] = make_double2((w[3].y - w[3].x) * r2, -(w[3].x + w[3].y) * r2);
      dft4(v[0], v[1], v[2], v[3]);
      dft4(w[0], w[1], w[2], w[3]);
      __syncthreads();  // previous FFT's reads of cbuf are done
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        cbuf[pidx(j * 8 + 2 * q)] = v[q];
        cbuf[pidx(j * 8 + 2 * q + 1)] = w[q];
      }
      __syncthreads();  // (also: every thread has read rows 2f, 2f+1)
      auto emit = [&](int k, double ya, double yb) {
        ra[k - 1] = ya;
        rb[k - 1] = yb;
      };
      if constexpr (last_radix<L>() == 4) {
        fft_middle_stages<L, kThreads>(cbuf, tw);
        last_radix4_stage_with_post<L, kThreads>(cbuf, tw, hs, nn, emit);
      } else {
        fft_after_first_stage<L, 1, kThreads>(cbuf, tw);
        for (int e = j; e < nn; e += kThreads) {
          const int k = e + 1;
          const double2 wk = cbuf[pidx(k)], wm = cbuf[pidx(L - k)];
          emit(k, -hs * (wk.y - wm.y), hs * (wk.x - wm.x));
        }
      }
    }
    __syncthreads();  // all G rows of results are in the stage buffer
    for (int e = threadIdx.x; e < G * nn; e += kThreads) {
      const int v = e % G, kk = e / G;
      const int64_t b = vbase[cur][v];
      if (b >= 0) __stcs(dst + b + int64_t(kk) * inner, st[v * RP + kk]);
    }
  }
  cp_async_wait<0>();
}

}  // namespace stkg
