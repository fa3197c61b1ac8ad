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
// 48 instead of 80 B/unknown.  The carries y_{l-1} of the tile's G n_0 modes stay on the
// SM (registers, or shared memory with CS): thread t of pair f owns the outputs
// e = t + T i - 1 (i < V) of its pair's two columns, reads g~ from the forward pass's
// OutPair staging and writes w y at the linear position e + 1 that the inverse
// pre-processing reads (tools/banksim: both conflict-free).  The next slice's tile is staged
// into its own buffer while the current slice computes (cp.async, or TMA boxes with TMA;
// the layout of dst_half_strided2_kernel: a swizzled mirror of the 16P-byte global rows).
//
// The per-step pivot is applied as y = (g - sub y) * r with r a Newton-refined reciprocal of
// piv = d_l + lambda c_l (two steps from rcp.approx: within an ulp of 1/piv; the reference
// divides) -- the kernel is bound by shared-memory traffic, and the ~25-instruction IEEE
// division per mode-step would double its FP64 issue.
#pragma once

#include "dst_half.cuh"

namespace stkg {

// CS: carries in shared memory (one double2 per slot) instead of registers; TMA: the tile is
// staged by SWIZZLE_64B TMA boxes (one elected thread, mbarrier) instead of per-thread
// cp.async (P = 4 only: 64-byte rows).
// VV: complex values per thread of the FFTs (16: radix-16,16,4 stages, 64 threads per pair for
// N = 1024; 8: radix-8,8,8,2 stages, 128 threads per pair -- twice the warps per SM for the
// same tile, one more shared-memory exchange per transform).
// MB: minimum resident CTAs per SM for __launch_bounds__ (2 caps registers at 128 so that
// other kernels' CTAs can share the SM -- the overlapped 2D schedule's contiguous passes).
template <int N, int PP, bool CS = false, bool TMA = false, int VV = half2_v<N>(), int MB = 1>
struct FusedCfg {
  using B = HalfStrided2Cfg<N, PP, true>;  // tile geometry (swizzle), region size
  static constexpr int V = VV, T = N / V, P = B::P, G = B::G, kThreads = P * T;
  static constexpr int kRegion = B::kRegion;
  static constexpr int kBoxRows = 256;
  static constexpr int kBoxes = (N - 1 + kBoxRows - 1) / kBoxRows;
  // bytes: regions | (512-byte aligned) tile | carries
  static constexpr size_t kRegionBytes = size_t(P) * kRegion * sizeof(double2);
  static constexpr size_t kTileBytes =
      TMA ? size_t(kBoxes) * kBoxRows * 64 : size_t(B::kTile) * sizeof(double2);
  static constexpr size_t kTileOff = TMA ? (kRegionBytes + 511) / 512 * 512 : kRegionBytes;
  static constexpr size_t kCarryOff = kTileOff + kTileBytes;
  // (the dynamic buffer is declared 1024-byte aligned, so kTileOff's 512-byte alignment is
  // the SWIZZLE_64B pattern's; kernels check the base at run time)
  // scan partials and the mbarrier live in the dynamic buffer too: with no static shared
  // memory the dynamic buffer starts at the (1024-byte aligned) start of the CTA's window
  static constexpr int kRedPer = T > 32 ? 2 * (T / 32) : 2;
  static constexpr size_t kRedOff = kCarryOff + (CS ? size_t(P) * N * sizeof(double2) : 0);
  static constexpr size_t kBarOff = kRedOff + size_t(P) * kRedPer * sizeof(double);
  static constexpr size_t kSmem = kBarOff + 16;
  static_assert(!TMA || P == 4, "TMA staging: tiles of 4 pairs (64-byte rows)");
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
// map (TMA only): S viewed as [ntc n_0 rows] x [inner columns], boxes of {8, 256}.
#define STKG_FUSED_PARAMS                                                                   \
  double *S, int64_t inner, int64_t slice, int64_t ntc, int64_t l0,                        \
      const double2 *__restrict__ tw2, double scale, const double *__restrict__ lam_ax,     \
      const double *__restrict__ w_ax, const double *__restrict__ lam_col,                  \
      const double *__restrict__ w_col, const double *__restrict__ d_diag,                  \
      const double *__restrict__ d_sup, const double *__restrict__ c_diag,                  \
      const double *__restrict__ c_sup, double *__restrict__ carry
#define STKG_FUSED_ARGS \
  S, inner, slice, ntc, l0, tw2, scale, lam_ax, w_ax, lam_col, w_col, d_diag, d_sup, c_diag, c_sup, carry

template <int N, int PP, bool CS, bool TMA, int VV, int MB>
__device__ __forceinline__ void heat_fused_axis0_body(const CUtensorMap& map, STKG_FUSED_PARAMS) {
  using C = FusedCfg<N, PP, CS, TMA, VV, MB>;
  using SC = typename C::B;
  using OP = OutPair<N, 4>;
  constexpr int V = C::V, T = C::T, P = C::P, n = N - 1, RG = C::kRegion;
  extern __shared__ __align__(1024) unsigned char fsraw[];
  unsigned char* sbase = fsraw;
  if constexpr (TMA) {  // the SWIZZLE_64B tile needs a 512-byte aligned destination
    if ((static_cast<unsigned>(__cvta_generic_to_shared(fsraw)) & 511u) != 0u) __trap();
  }
  double2* sreg = reinterpret_cast<double2*>(sbase);
  double2* stile = reinterpret_cast<double2*>(sbase + C::kTileOff);
  double* red = reinterpret_cast<double*>(sbase + C::kRedOff);  // [P][kRedPer]
  uint64_t& mbar = *reinterpret_cast<uint64_t*>(sbase + C::kBarOff);
  const int f = threadIdx.x / T, t = threadIdx.x % T;
  const int bar = P > 1 ? 1 + f : 0;
  double2* region = sreg + f * RG;
  double2* creg = reinterpret_cast<double2*>(sbase + C::kCarryOff) + f * N;  // CS only
  const int64_t i0 = int64_t(blockIdx.x) * C::G;
  const int64_t ca = i0 + 2 * f;  // this pair's columns ca, ca + 1
  const double hs = 0.5 * scale;
  const double lca = lam_col[ca], lcb = lam_col[ca + 1];
  const double wca = w_col[ca], wcb = w_col[ca + 1];

  auto load_tile = [&](int64_t j) {  // local slice j of this launch
    if constexpr (TMA) {
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive_expect_tx(&mbar, static_cast<unsigned>(C::kTileBytes));
#pragma unroll
        for (int b = 0; b < C::kBoxes; ++b)
          tma_load_2d(reinterpret_cast<char*>(stile) + b * C::kBoxRows * 64, &map,
                      static_cast<int>(i0), static_cast<int>(j * n + b * C::kBoxRows), &mbar);
      }
    } else {
      const double* src = S + j * slice + i0;
      for (int e = threadIdx.x; e < P * n; e += C::kThreads) {
        const int c = e % P, r = e / P;
        cp_async16(stile + r * P + SC::chunk(r, c), src + int64_t(r) * inner + 2 * c);
      }
      cp_async_commit();
    }
  };

  // The recurrence's slots: thread t handles the outputs e = t + T i - 1 (i < V; e = -1 is
  // no output): read from OutPair<N, 4> (8 consecutive e of a quarter-warp fall in 8
  // distinct bank groups), written as y at the linear position e + 1 that the inverse
  // pre-processing reads (x_m at m, x_{N-m} at N - m: consecutive, conflict-free).
  double ya[CS ? 1 : V], yb[CS ? 1 : V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int e = t + T * i - 1;
    const double a = (l0 > 0 && e >= 0) ? carry[int64_t(e) * inner + ca] : 0.0;
    const double b = (l0 > 0 && e >= 0) ? carry[int64_t(e) * inner + ca + 1] : 0.0;
    if constexpr (CS) {
      creg[t + T * i] = make_double2(a, b);
    } else {
      ya[i] = a;
      yb[i] = b;
    }
  }
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(&mbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
  }
  unsigned phase = 0;

  if (ntc > 0) load_tile(0);
  for (int64_t j = 0; j < ntc; ++j) {
    const int64_t l = l0 + j;
    if constexpr (TMA) {
      mbar_wait(&mbar, phase);
      phase ^= 1u;
    } else {
      cp_async_wait<0>();
    }
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
    half_fft_post<N, V>(x, region, tw2, t, hs, red + f * C::kRedPer, OP{region}, bar);
    fft_sync<T>(bar);

    // recurrence (stk/sylvester.hpp:131-139): y = (g~ - sub y) / piv per mode
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int e = t + T * i - 1;
      x[i] = e >= 0 ? region[OP::idx(e)] : make_double2(0.0, 0.0);
    }
    fft_sync<T>(bar);  // every slot was read: the linear y may overwrite the region
    const double dd = __ldg(d_diag + l), cd = __ldg(c_diag + l);
    const double ds = l > 0 ? __ldg(d_sup + l - 1) : 0.0, cs = l > 0 ? __ldg(c_sup + l - 1) : 0.0;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int e = t + T * i - 1;
      if (e >= 0) {
        const double le = __ldg(lam_ax + e), we = __ldg(w_ax + e);
        const double la = le + lca, lb = le + lcb;
        const double ra = nr_recip(dd + la * cd), rb = nr_recip(dd + lb * cd);
        double pa, pb;
        if constexpr (CS) {
          const double2 c2 = creg[t + T * i];
          pa = c2.x;
          pb = c2.y;
        } else {
          pa = ya[i];
          pb = yb[i];
        }
        const double na = (x[i].x - (ds + la * cs) * pa) * ra;
        const double nb = (x[i].y - (ds + lb * cs) * pb) * rb;
        if constexpr (CS) {
          creg[t + T * i] = make_double2(na, nb);
        } else {
          ya[i] = na;
          yb[i] = nb;
        }
        x[i] = make_double2(we * wca * na, we * wcb * nb);
        region[t + T * i] = x[i];
      }
    }
    fft_sync<T>(bar);

    // inverse transform along axis 0 (DST-I is its own inverse): this thread's own y at
    // m = t + T p is x[p] already (e = m - 1); only the mirrored y at N - m comes from the
    // linear layout
#pragma unroll
    for (int p = 0; p < V; ++p) {
      const int m = t + T * p;
      const double2 u = x[p];
      x[p] = make_double2(0.0, 0.0);
      if (m > 0) {
        const double s = -__ldg(&tw2[m].y);
        const double2 w = region[N - m];
        x[p] = half_pre(s, u.x, w.x, u.y, w.y);
      }
    }
    half_fft_post<N, V>(x, region, tw2, t, hs, red + f * C::kRedPer, OP{region}, bar);
    __syncthreads();
    double* dst = S + j * slice + i0;
    for (int e = threadIdx.x; e < P * n; e += C::kThreads) {
      const int q = e % P, kk = e / P;
      __stcs(reinterpret_cast<double2*>(dst + int64_t(kk) * inner + 2 * q),
             sreg[q * RG + OP::idx(kk)]);
    }
  }
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int e = t + T * i - 1;
    if (e >= 0) {
      double a, b;
      if constexpr (CS) {
        const double2 c2 = creg[t + T * i];
        a = c2.x;
        b = c2.y;
      } else {
        a = ya[i];
        b = yb[i];
      }
      carry[int64_t(e) * inner + ca] = a;
      carry[int64_t(e) * inner + ca + 1] = b;
    }
  }
}



template <int N, int PP, bool CS, bool TMA, int VV, int MB>
__global__ void __launch_bounds__(FusedCfg<N, PP, CS, TMA, VV, MB>::kThreads,
                                  FusedCfg<N, PP, CS, TMA, VV, MB>::kThreads >= 256
                                      ? MB : 256 / FusedCfg<N, PP, CS, TMA, VV, MB>::kThreads)
    heat_fused_axis0_kernel(const __grid_constant__ CUtensorMap map, STKG_FUSED_PARAMS) {
  heat_fused_axis0_body<N, PP, CS, TMA, VV, MB>(map, STKG_FUSED_ARGS);
}

}  // namespace stkg
