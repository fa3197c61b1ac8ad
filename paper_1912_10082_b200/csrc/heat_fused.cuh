// Time-marching fused pass of the P1_DST padded device solve (K2b + K3 in one kernel).
//
// run_chunk_padded's five HBM passes are  F -(fastest axis)-> S -(other axes)-> S -(scan)->
// S -(other axes)-> S -(fastest axis)-> U.  The recurrence of solve_projected_heat_with
// (stk/sylvester.hpp:128-140) is independent per mode and sequential in time, and the slowest
// spatial axis's forward and inverse transforms are independent per time slice, so one CTA
// can own a tile of G = 2P neighbouring columns of axis 0 (all n_0 rows) and march through
// the time slices:
//
//     for l in slices:  tile_l  -(forward DST-I along axis 0)->  g~  -(recurrence, carries
//                       in registers)->  w y  -(inverse DST-I along axis 0)->  tile_l
//
// The modal data never leaves the CTA between the three steps, so the scan's HBM pass and
// the second strided pass disappear: 3 HBM passes per 2D solve (5 in 3D) instead of 5 (7),
// 48 instead of 80 B/unknown.  The carries y_{l-1} of the tile's G n_0 modes live in
// registers: thread t of pair f owns the OutPair staging slots s = t + T i (i < V), which
// cover the tile's two columns' n_0 modes exactly once (the even half of OutPair holds
// k < N/2 for e = 2k, the odd half e = 2k - 1), and the quarter-warp reads of consecutive
// slots are bank-conflict free.  The next slice's tile is staged by 16-byte cp.async into
// its own buffer while the current slice computes (the layout of dst_half_strided2_kernel:
// a swizzled mirror of the 16P-byte global rows).
//
// The per-step pivot is applied as y = (g - sub y) * r with r a Newton-refined reciprocal of
// piv = d_l + lambda c_l (two steps from rcp.approx: within an ulp of 1/piv; the reference
// divides) -- the kernel is bound by shared-memory traffic, and the ~25-instruction IEEE
// division per mode-step would double its FP64 issue.
#pragma once

#include "dst_half.cuh"

namespace stkg {

template <int N, int PP>
struct FusedCfg {
  using B = HalfStrided2Cfg<N, PP, true>;  // pair regions + separate staged tile
  static constexpr int V = B::V, T = B::T, P = B::P, G = B::G, kThreads = B::kThreads;
  static constexpr int kRegion = B::kRegion, kTileOff = B::kTileOff;
  static constexpr size_t kSmem = B::kSmem;
};

template <int N>
constexpr int fused_pairs() { return half2_pairs<N>(); }

__device__ __forceinline__ double nr_recip(double p) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
  double e = fma(-p, r, 1.0);
  r = fma(r, e, r);
  e = fma(-p, r, 1.0);
  return fma(r, e, r);
}

// S: the padded scratch (slice stride `slice` = n_0 * inner doubles), modified in place.
// Tile `blockIdx.x` = columns [G b, G b + G) of every slice.  lam_ax / w_ax: axis-0
// eigenvalues and 1/mu weights (n_0 entries); lam_col / w_col: the summed eigenvalue and the
// weight product of the faster axes for each column (inner entries; pad lane 0 / 0).
// carry (slice entries, indexed like one slice): y_{l0-1} in, y_{l0+ntc-1} out.
template <int N, int PP>
__global__ void __launch_bounds__(FusedCfg<N, PP>::kThreads,
                                  FusedCfg<N, PP>::kThreads >= 256 ? 1 : 256 / FusedCfg<N, PP>::kThreads)
    heat_fused_axis0_kernel(double* S, int64_t inner, int64_t slice, int64_t ntc, int64_t l0,
                            const double2* __restrict__ tw2, double scale,
                            const double* __restrict__ lam_ax, const double* __restrict__ w_ax,
                            const double* __restrict__ lam_col, const double* __restrict__ w_col,
                            const double* __restrict__ d_diag, const double* __restrict__ d_sup,
                            const double* __restrict__ c_diag, const double* __restrict__ c_sup,
                            double* __restrict__ carry) {
  using C = FusedCfg<N, PP>;
  using SC = typename C::B;
  constexpr int V = C::V, T = C::T, P = C::P, n = N - 1, RG = C::kRegion, H2 = N / 2;
  extern __shared__ __align__(128) double2 sreg[];
  __shared__ double red[P][T > 32 ? 2 * (T / 32) : 2];
  const int f = threadIdx.x / T, t = threadIdx.x % T;
  const int bar = P > 1 ? 1 + f : 0;
  double2* region = sreg + f * RG;
  double2* stile = sreg + C::kTileOff;
  const int64_t i0 = int64_t(blockIdx.x) * C::G;
  const int64_t ca = i0 + 2 * f;  // this pair's columns ca, ca + 1
  const double hs = 0.5 * scale;
  const double lca = lam_col[ca], lcb = lam_col[ca + 1];
  const double wca = w_col[ca], wcb = w_col[ca + 1];

  auto load_tile = [&](int64_t l) {
    const double* src = S + l * slice + i0;
    for (int e = threadIdx.x; e < P * n; e += C::kThreads) {
      const int c = e % P, r = e / P;
      cp_async16(stile + r * P + SC::chunk(r, c), src + int64_t(r) * inner + 2 * c);
    }
    cp_async_commit();
  };
  // slot s = t + T i of this pair's OutPair staging -> output index e (-1: the unused odd
  // slot k = 0).  With T a multiple of 64 the swizzle of kk = t + T i' depends on t only,
  // so e is 2 k0 + 2 T i' (- 1): constant offsets from one base (fewer live registers).
  const int k0 = t ^ ((t >> 3) & 7);
  auto slot_e = [&](int i) {
    const int ih = i % (V / 2);
    int k;
    if constexpr (T % 64 == 0) {
      k = k0 + T * ih;
    } else {
      const int kk = t + T * ih;
      k = kk ^ ((kk >> 3) & 7);
    }
    return i >= V / 2 ? (k == 0 ? -1 : 2 * k - 1) : 2 * k;
  };
  static_assert(T * V / 2 == H2, "slots i < V/2 are the even half of OutPair");

  double ya[V], yb[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int e = slot_e(i);
    ya[i] = (l0 > 0 && e >= 0) ? carry[int64_t(e) * inner + ca] : 0.0;
    yb[i] = (l0 > 0 && e >= 0) ? carry[int64_t(e) * inner + ca + 1] : 0.0;
  }

  if (ntc > 0) load_tile(0);
  for (int64_t j = 0; j < ntc; ++j) {
    const int64_t l = l0 + j;
    cp_async_wait<0>();
    __syncthreads();  // tile j landed; the previous slice's stores have read the regions
    double2 x[V];
#pragma unroll
    for (int p = 0; p < V; ++p) {
      const int m = t + T * p;
      x[p] = make_double2(0.0, 0.0);
      if (m > 0) {
        const int r0 = m - 1, r1 = N - m - 1;
        const double s = -__ldg(&tw2[m].y);
        const double2 u = stile[r0 * P + SC::chunk(r0, f)], w = stile[r1 * P + SC::chunk(r1, f)];
        x[p] = half_pre(s, u.x, w.x, u.y, w.y);
      }
    }
    __syncthreads();  // every pair has read the tile: stage the next slice's
    if (j + 1 < ntc) load_tile(j + 1);

    // forward transform along axis 0 -> OutPair (g~ of both columns, unweighted)
    half_fft_post<N, V>(x, region, tw2, t, hs, red[f], OutPair<N>{region}, bar);
    fft_sync<T>(bar);

    // recurrence (stk/sylvester.hpp:131-139) on this thread's slots, in place
    const double dd = __ldg(d_diag + l), cd = __ldg(c_diag + l);
    const double ds = l > 0 ? __ldg(d_sup + l - 1) : 0.0, cs = l > 0 ? __ldg(c_sup + l - 1) : 0.0;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int s = t + T * i;
      const int e = slot_e(i);
      if (e >= 0) {
        const double le = __ldg(lam_ax + e), we = __ldg(w_ax + e);
        const double la = le + lca, lb = le + lcb;
        const double2 g = region[s];
        const double ra = nr_recip(dd + la * cd), rb = nr_recip(dd + lb * cd);
        ya[i] = (g.x - (ds + la * cs) * ya[i]) * ra;
        yb[i] = (g.y - (ds + lb * cs) * yb[i]) * rb;
        region[s] = make_double2(we * wca * ya[i], we * wcb * yb[i]);
      }
    }
    fft_sync<T>(bar);

    // inverse transform along axis 0 (DST-I is its own inverse) from OutPair
    const OutPair<N> op{region};
#pragma unroll
    for (int p = 0; p < V; ++p) {
      const int m = t + T * p;
      x[p] = make_double2(0.0, 0.0);
      if (m > 0) {
        const double s = -__ldg(&tw2[m].y);
        double ua, ub, wa, wb;
        op.get(m - 1, ua, ub);
        op.get(N - m - 1, wa, wb);
        x[p] = half_pre(s, ua, wa, ub, wb);
      }
    }
    half_fft_post<N, V>(x, region, tw2, t, hs, red[f], OutPair<N>{region}, bar);
    __syncthreads();
    double* dst = S + j * slice + i0;
    for (int e = threadIdx.x; e < P * n; e += C::kThreads) {
      const int q = e % P, kk = e / P;
      __stcs(reinterpret_cast<double2*>(dst + int64_t(kk) * inner + 2 * q),
             sreg[q * RG + OutPair<N>::idx(kk)]);
    }
  }
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int e = slot_e(i);
    if (e >= 0) {
      carry[int64_t(e) * inner + ca] = ya[i];
      carry[int64_t(e) * inner + ca + 1] = yb[i];
    }
  }
}

}  // namespace stkg
