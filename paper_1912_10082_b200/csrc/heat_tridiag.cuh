// Time-marching line-solve pass over axis 0 of the P1_DST padded device solve (K2e).
//
// solve_projected_heat_with (stk/sylvester.hpp:117-142) diagonalises every spatial axis and
// runs the temporal recurrence per mode.  For a uniform P1 axis the mass and stiffness
// factors M_0 = tridiag(m_o, m_d, m_o), A_0 = tridiag(a_o, a_d, a_o) are Toeplitz, so axis 0
// need not be transformed at all: with the faster axes diagonalised (column c: eigenvalue sum
// lambda_c, weight w_c = prod 1/mu), the step l of the recurrence is, per column, one
// symmetric tridiagonal solve along axis 0 (the identity Q diag(mu) Q = M_0,
// Q diag(mu lambda) Q = A_0 applied to the modal recurrence of heat_fused.cuh):
//
//     T z_l = w_c g_l - T' z_{l-1},   T  = (d_l + lambda_c c_l) M_0 + c_l A_0
//                                     T' = (d^s_{l-1} + lambda_c c^s_{l-1}) M_0 + c^s_{l-1} A_0
//
// z_l is exactly what heat_fused_axis0_kernel writes (inverse transform of the weighted modal
// solution), with O(n) instead of O(n log n) work per column and two shared-memory accesses
// per value instead of two FFTs' worth: the pass becomes an HBM stream.
//
// Two kernels:
//  * heat_tridiag_tma_kernel (the default; second half of this file): TMA tile loads and
//    stores, the solve as constant-coefficient causal / anti-causal sweeps (method of images
//    for the Toeplitz tridiagonal: no per-row data at all), uniform or non-uniform time grids;
//  * heat_tridiag_axis0_kernel (STKG_TRI_V=0; the first version, kept as an independent
//    cross-check): cp.async staging, the solve as an LDL^T chunked scan whose reciprocal
//    pivots 1/w_i are computed once per plan (tri_factor_kernel) and held in registers;
//    uniform time grids only.  Described next.
//
// LDL^T kernel.  One CTA owns G = 2P neighbouring columns of axis 0 (all n_0 rows) and marches
// through the time slices.  T = N/16 threads share a column pair; thread t holds rows
// 16t .. 16t+15 of both columns.  The two triangular solves are first-order linear recurrences
// along the rows, run as a chunked scan: every thread runs its 16 rows with zero carry-in, the
// chunk end values are combined across the T threads by a Kogge-Stone scan whose weights
// (products of the chunks' multipliers) are per-plan constants in registers, and every thread
// reruns its rows from its carry-in.  No division, no transform, z_{l-1} stays in registers.
// Tiles are staged by 16-byte cp.async into ST buffers (two slices in flight while one is
// solved); a 16-row block of the tile is followed by 16 bytes of skew so that the 8 threads
// of a quarter-warp (row chunks 16 rows apart) read 8 distinct bank groups.
#pragma once

#include "dst_half.cuh"

namespace stkg {

constexpr int tri_ilog2(int v) { return v <= 1 ? 0 : 1 + tri_ilog2(v / 2); }

template <int N, int PP, int ST = 3>
struct TriCfg {
  static constexpr int R = 16, T = N / R, P = PP, G = 2 * PP, kThreads = PP * T, n = N - 1;
  static constexpr int W = T < 32 ? T : 32;  // lanes of one scan segment
  static constexpr int LW = tri_ilog2(W);
  static constexpr int kBlk = R * P + 1;   // double2 per 16-row block (+ 16 bytes of skew)
  static constexpr int kBuf = T * kBlk;    // double2 per tile buffer (N rows: one phantom)
  static constexpr int kStages = ST;
  static constexpr size_t kXchOff = size_t(ST) * kBuf * sizeof(double2);
  static constexpr size_t kSmem = kXchOff + size_t(P) * 4 * sizeof(double2);
  static_assert(T >= 2 && (T <= 32 || T == 64), "2..32 lanes or two warps per column pair");
  static_assert(kThreads % 32 == 0 && kThreads <= 1024, "whole warps");
  static_assert(size_t(2 * T) * P * sizeof(double2) <= size_t(ST) * kBuf * sizeof(double2),
                "the prologue's multiplier products fit the tile buffers");
};

// Reciprocal pivots of T_c = tridiag(a, b, a) for every column c (Thomas / LDL^T without
// pivoting: w_0 = b, w_i = b - a^2 / w_{i-1}), stored as iw[i * inner + c] for i < n and 0 at
// the phantom row i = n.  *bad is set when a pivot is not positive (T_c not SPD: the caller
// keeps the transform-based pass).
__global__ void tri_factor_kernel(double* __restrict__ iw, int64_t inner, int n,
                                  const double* __restrict__ lam_col, double dd, double cd,
                                  double md, double mo, double ad, double ao, int* bad) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= inner) return;
  const double p = dd + lam_col[c] * cd;
  const double a = p * mo + cd * ao, b = p * md + cd * ad, a2 = a * a;
  double w = b;
  bool ok = true;
  for (int i = 0; i < n; ++i) {
    ok = ok && (w > 0.0) && (w <= 1.7976931348623157e308);
    const double r = 1.0 / w;
    iw[int64_t(i) * inner + c] = r;
    w = b - a2 * r;
  }
  iw[int64_t(n) * inner + c] = 0.0;
  if (!ok) atomicOr(bad, 1);
}

__device__ __forceinline__ double2 shfl_up2(double2 v, int d, int w) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, d, w), __shfl_up_sync(0xffffffffu, v.y, d, w));
}
__device__ __forceinline__ double2 shfl_down2(double2 v, int d, int w) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, d, w),
                      __shfl_down_sync(0xffffffffu, v.y, d, w));
}

// S: the padded scratch (slice stride `slice` = n_0 * inner doubles), modified in place.
// Tile blockIdx.x = columns [G b, G b + G) of every slice.  iw: tri_factor_kernel's output.
// dd, cd: the temporal diagonals (every step); ds, cs: the sub-diagonals (steps l > 0).
// carry (slice entries, indexed like one slice): z_{l0-1} in (read when l0 > 0),
// z_{l0+ntc-1} out.
template <int N, int PP, int ST>
__global__ void __launch_bounds__(TriCfg<N, PP, ST>::kThreads, 1)
    heat_tridiag_axis0_kernel(double* S, int64_t inner, int64_t slice, int64_t ntc, int64_t l0,
                              const double* __restrict__ iw, const double* __restrict__ lam_col,
                              const double* __restrict__ w_col, double dd, double ds, double cd,
                              double cs, double md, double mo, double ad, double ao,
                              double* __restrict__ carry) {
  using C = TriCfg<N, PP, ST>;
  constexpr int R = C::R, T = C::T, P = C::P, n = C::n, W = C::W, LW = C::LW;
  extern __shared__ __align__(16) unsigned char triraw[];
  double2* bufs = reinterpret_cast<double2*>(triraw);
  double2* xch = reinterpret_cast<double2*>(triraw + C::kXchOff);  // [P][4]
  const int tid = threadIdx.x;
  const int f = tid / T, t = tid % T;
  const int sl = t & (W - 1);            // lane within the scan segment
  const int bar = 1 + f;                 // the pair's named barrier (T == 64)
  const int64_t i0 = int64_t(blockIdx.x) * C::G;
  const int64_t ca = i0 + 2 * f;
  const int row0 = R * t;

  // per-column constants: T = tridiag(ta, ., ta) (the diagonal is inside the pivots),
  // T' = tridiag(sa, sb, sa), load weight wc
  double2 ta, sa, sb, wc;
  {
    const double la = lam_col[ca], lb = lam_col[ca + 1];
    const double pa = dd + la * cd, pb = dd + lb * cd;
    ta = make_double2(pa * mo + cd * ao, pb * mo + cd * ao);
    const double qa = ds + la * cs, qb = ds + lb * cs;
    sa = make_double2(qa * mo + cs * ao, qb * mo + cs * ao);
    sb = make_double2(qa * md + cs * ad, qb * md + cs * ad);
    wc = make_double2(w_col[ca], w_col[ca + 1]);
  }
  // reciprocal pivots of rows row0 - 1 .. row0 + 15 (0 above the first row)
  double2 iv[R + 1];
#pragma unroll
  for (int k = 0; k <= R; ++k) {
    const int r = row0 - 1 + k;
    iv[k] = r >= 0 ? *reinterpret_cast<const double2*>(iw + int64_t(r) * inner + ca)
                   : make_double2(0.0, 0.0);
  }
  // scan weights: products of the chunks' multipliers.  Forward chunk u maps its carry-in by
  // Pf_u = prod_j (-ta iw_{16u+j-1}); backward by Pb_u = prod_j (-ta iw_{16u+j}).
  double2 wf[LW], wb[LW], wfx = make_double2(0.0, 0.0), wbx = make_double2(0.0, 0.0);
  {
    double2 pf = make_double2(1.0, 1.0), pb = make_double2(1.0, 1.0);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      pf.x *= -ta.x * iv[k].x;
      pf.y *= -ta.y * iv[k].y;
      pb.x *= -ta.x * iv[k + 1].x;
      pb.y *= -ta.y * iv[k + 1].y;
    }
    double2* sp = bufs;  // [P][2][T], before any tile is staged
    sp[(f * 2 + 0) * T + t] = pf;
    sp[(f * 2 + 1) * T + t] = pb;
    __syncthreads();
    const double2* spf = sp + (f * 2 + 0) * T;
    const double2* spb = sp + (f * 2 + 1) * T;
#pragma unroll
    for (int k = 0; k < LW; ++k) {
      const int d = 1 << k;
      double2 a = make_double2(0.0, 0.0), b = make_double2(0.0, 0.0);
      if (sl >= d) {
        a = make_double2(1.0, 1.0);
        for (int u = t - d + 1; u <= t; ++u) a.x *= spf[u].x, a.y *= spf[u].y;
      }
      if (sl + d < W) {
        b = make_double2(1.0, 1.0);
        for (int u = t; u < t + d; ++u) b.x *= spb[u].x, b.y *= spb[u].y;
      }
      wf[k] = a;
      wb[k] = b;
    }
    if constexpr (T > 32) {
      if (t >= 32) {
        wfx = make_double2(1.0, 1.0);
        for (int u = 32; u <= t; ++u) wfx.x *= spf[u].x, wfx.y *= spf[u].y;
      } else {
        wbx = make_double2(1.0, 1.0);
        for (int u = t; u < 32; ++u) wbx.x *= spb[u].x, wbx.y *= spb[u].y;
      }
    }
    __syncthreads();  // the products were read: the buffers may be staged
  }

  auto tile_at = [&](int st, int r, int c) -> double2* {
    return bufs + st * C::kBuf + (r >> 4) * C::kBlk + (r & 15) * P + c;
  };
  auto load_tile = [&](int64_t j, int st) {
    const double* src = S + j * slice + i0;
    for (int e = tid; e < P * n; e += C::kThreads) {
      const int c = e % P, r = e / P;
      cp_async16(tile_at(st, r, c), src + int64_t(r) * inner + 2 * c);
    }
  };
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < ntc) load_tile(s, s);
    cp_async_commit();
  }

  // z_{l0-1}: this thread's rows, the row above its first (zu) and below its last (zn)
  double2 x[R], zn = make_double2(0.0, 0.0), zu = make_double2(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int r = row0 + k;
    x[k] = (l0 > 0 && r < n) ? *reinterpret_cast<const double2*>(carry + int64_t(r) * inner + ca)
                             : make_double2(0.0, 0.0);
  }
  if (l0 > 0) {
    if (row0 > 0) zu = *reinterpret_cast<const double2*>(carry + int64_t(row0 - 1) * inner + ca);
    if (row0 + R < n) zn = *reinterpret_cast<const double2*>(carry + int64_t(row0 + R) * inner + ca);
  }
  const bool phantom_owner = t == T - 1;  // its last row (index n) is not in the matrix

  for (int64_t j = 0; j < ntc; ++j) {
    const int st = static_cast<int>(j % ST);
    cp_async_wait<ST - 2>();
    __syncthreads();  // tile j landed; the copy-out of slice j - 1 has read its buffer
    if (j + ST - 1 < ntc) load_tile(j + ST - 1, static_cast<int>((j + ST - 1) % ST));
    cp_async_commit();

    // right-hand side in place: r_i = w_c g_i - sb z_i - sa (z_{i-1} + z_{i+1})
    if (j > 0) {
      zu = shfl_up2(x[R - 1], 1, W);
      if (sl == 0) zu = (T > 32 && t == 32) ? xch[f * 4 + 2] : make_double2(0.0, 0.0);
    }
    {
      const double2* tb = tile_at(st, row0, f);
      double2 zl = zu;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const double2 g = tb[k * P];
        const double2 zc = x[k];
        const double2 zr = k + 1 < R ? x[k + 1] : zn;
        const double ra = fma(sb.x, zc.x, sa.x * (zl.x + zr.x));
        const double rb = fma(sb.y, zc.y, sa.y * (zl.y + zr.y));
        x[k] = make_double2(fma(wc.x, g.x, -ra), fma(wc.y, g.y, -rb));
        zl = zc;
      }
      if (phantom_owner) x[R - 1] = make_double2(0.0, 0.0);
    }

    // forward substitution f_i = r_i - (ta iw_{i-1}) f_{i-1}: chunk end with zero carry-in,
    // scan over the chunks, rerun from the carry-in
    double2 e = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      e.x = fma(-(ta.x * iv[k].x), e.x, x[k].x);
      e.y = fma(-(ta.y * iv[k].y), e.y, x[k].y);
    }
#pragma unroll
    for (int k = 0; k < LW; ++k) {
      const double2 v = shfl_up2(e, 1 << k, W);
      e.x = fma(wf[k].x, v.x, e.x);  // wf = 0 where the segment has no lane 2^k below
      e.y = fma(wf[k].y, v.y, e.y);
    }
    double2 lo = make_double2(0.0, 0.0);
    if constexpr (T > 32) {
      if (t == 31) xch[f * 4 + 0] = e;
      fft_sync<T>(bar);
      if (t >= 32) {
        lo = xch[f * 4 + 0];  // f at the end of chunk 31
        e.x = fma(wfx.x, lo.x, e.x);
        e.y = fma(wfx.y, lo.y, e.y);
      }
    }
    {
      double2 fc = shfl_up2(e, 1, W);
      if (sl == 0) fc = lo;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        fc.x = fma(-(ta.x * iv[k].x), fc.x, x[k].x);
        fc.y = fma(-(ta.y * iv[k].y), fc.y, x[k].y);
        x[k] = fc;
      }
    }

    // back substitution z_i = iw_i (f_i - ta z_{i+1}), the same way from the last row up
    e = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = R - 1; k >= 0; --k) {
      e.x = iv[k + 1].x * fma(-ta.x, e.x, x[k].x);
      e.y = iv[k + 1].y * fma(-ta.y, e.y, x[k].y);
    }
#pragma unroll
    for (int k = 0; k < LW; ++k) {
      const double2 v = shfl_down2(e, 1 << k, W);
      e.x = fma(wb[k].x, v.x, e.x);  // wb = 0 where the segment has no lane 2^k above
      e.y = fma(wb[k].y, v.y, e.y);
    }
    double2 hi = make_double2(0.0, 0.0);
    if constexpr (T > 32) {
      if (t == 32) xch[f * 4 + 1] = e;
      fft_sync<T>(bar);
      if (t < 32) {
        hi = xch[f * 4 + 1];  // z of the first row of chunk 32
        e.x = fma(wbx.x, hi.x, e.x);
        e.y = fma(wbx.y, hi.y, e.y);
      }
    }
    zn = shfl_down2(e, 1, W);  // z of the row below this chunk: also the next step's neighbour
    if (sl == W - 1) zn = hi;
    {
      double2 zc = zn;
#pragma unroll
      for (int k = R - 1; k >= 0; --k) {
        zc.x = iv[k + 1].x * fma(-ta.x, zc.x, x[k].x);
        zc.y = iv[k + 1].y * fma(-ta.y, zc.y, x[k].y);
        x[k] = zc;
      }
    }
    {
      double2* tb = tile_at(st, row0, f);
#pragma unroll
      for (int k = 0; k < R; ++k) tb[k * P] = x[k];
    }
    if constexpr (T > 32) {
      if (t == 31) xch[f * 4 + 2] = x[R - 1];  // the next step's row above chunk 32
    }
    __syncthreads();
    double* dst = S + j * slice + i0;
    for (int q = tid; q < P * n; q += C::kThreads) {
      const int c = q % P, r = q / P;
      __stcs(reinterpret_cast<double2*>(dst + int64_t(r) * inner + 2 * c), *tile_at(st, r, c));
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int r = row0 + k;
    if (r < n) *reinterpret_cast<double2*>(carry + int64_t(r) * inner + ca) = x[k];
  }
}


// ---------------------------------------------------------------------------------------
// TMA variant (the default): the tile of slice j is loaded by cp.async.bulk.tensor boxes into
// one of two input buffers (full / empty mbarriers; the load of slice j + 2 is issued as soon
// as every thread has read slice j's tile, early in step j, so two slices are in flight) and
// the solved tile leaves from an output buffer by a bulk tensor store; no thread copies data.
// The tensor map views the launch's slices as [ntc][n_0 rows][inner columns]: rows past n_0
// are zero-filled on load and clipped on store, so the phantom rows need no special case.
// A thread owns R = 17 rows (odd): rows 17 t + k of 8 consecutive t differ in their low three
// bits, so TMA's own SWIZZLE_64B / SWIZZLE_128B row mirrors are read and written
// bank-conflict free (with 16-row chunks every lane of a quarter-warp would hit one bank group).
#ifndef STKG_TRI_PF
#define STKG_TRI_PF 0  // L2 prefetch distance of the line-solve pass in slices (<= 2: off;
                       // measured on cfg3: 3 neutral within noise, 5 and 8 slower)
#endif

template <int N, int PP>
struct TriTmaCfg {
  static constexpr int R = 17, T = N / 16, P = PP, G = 2 * PP, kThreads = PP * T, n = N - 1;
  static constexpr int W = T < 32 ? T : 32, LW = tri_ilog2(W);
  static constexpr int CW = P >= 8 ? 128 : 64;          // bytes per smem row of one column box
  static constexpr int CPB = CW / 16;                   // column pairs per column box
  static constexpr int NCB = P / CPB;                   // column boxes
  static constexpr int BR = N < 256 ? N : 256;          // rows per TMA box
  static constexpr int NRB = N / BR;                    // row boxes
  static constexpr int kRows = (T * R + 7) / 8 * 8;     // buffer rows (every lane's chunk)
  static constexpr int kBufBytes = NCB * kRows * CW;    // one tile buffer
  static constexpr unsigned kTxBytes = unsigned(NCB) * NRB * BR * CW;
  static constexpr size_t kXchOff = size_t(3) * kBufBytes;
  static constexpr size_t kBarOff = kXchOff + size_t(P) * 8 * sizeof(double2);
  static constexpr size_t kSmem = kBarOff + 8 * sizeof(uint64_t);
  static_assert(P == 4 || P % 8 == 0, "64-byte rows or whole 128-byte column boxes");
  static_assert(T >= 2 && (T <= 32 || T == 64), "2..32 lanes or two warps per column pair");
  static_assert(T * R >= N, "the chunks cover every row");
  static_assert(kBufBytes % 1024 == 0, "buffers keep the swizzle pattern's alignment");
};

__device__ __forceinline__ void tma_load_3d(void* smem, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(s),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(b)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int c0, int c1, int c2,
                                             const void* smem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(s)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}

// q^e for an integer e >= 0 (q may be negative or zero; 0^0 = 1).
__device__ __forceinline__ double tri_ipow(double q, int e) {
  double r = 1.0;
  while (e > 0) {
    if (e & 1) r *= q;
    q *= q;
    e >>= 1;
  }
  return r;
}

// The solve itself uses the Toeplitz structure once more: T = tridiag(a, b, a) is the
// restriction of the bi-infinite Toeplitz operator T_inf = L D L^T (constant pivot
// w = (b + sqrt(b^2 - 4 a^2)) / 2, multiplier m = a / w, |m| < 1) to odd, 2N-periodic
// sequences (method of images: the Dirichlet rows 0 and N are the mirror points).  With
// q = -m and gamma = 1 / sqrt(b^2 - 4 a^2), T_inf^{-1} is the convolution with
// gamma q^|k|, i.e. one causal and one anti-causal first-order recurrence with the CONSTANT
// coefficient q:
//     A_i = r_i + q A_{i-1},   B_i = r_i + q B_{i+1},   z_i = gamma (A_i + q B_{i+1})
// whose start values follow from the two zero-start totals a_N = sum_j q^{N-j} r_j and
// b_0 = sum_j q^j r_j:  A_0 = (q^N a_N - b_0) / (1 - q^{2N}),  B_N = -(q^N A_0 + a_N).
// So no per-row pivots are stored at all (the LDL^T variant above keeps 17 reciprocal pivots
// per column in registers); both zero-start recurrences and both chunk scans run side by
// side, one barrier per step joins the two warps of a column pair, and r is recovered from
// A in the second sweep (r_i = A_i - q A_{i-1}), so one register array holds z, r, A and z
// again.
// UNI: uniform time grid -- (dd, ds, cd, cs) are the temporal coefficients of every step and
// the per-column constants are set up once.  !UNI: the coefficients of step l come from the
// plan's bidiagonal arrays (the scalar arguments are unused) and the per-column constants
// (q, gamma, the chunk / image powers of q) are recomputed at the top of every step.
// GUARD: every row update is predicated on the row being real (k < cnt) on top of the
// phantom-row neutralisation.  The guards cost 450 instructions per warp and step and are
// redundant arithmetically, but plans with a full wave of tiles (cfg3: 128) run FASTER with
// them (3.0 vs 3.3 ms per launch, same box, alternating runs): the longer step keeps the
// demand just under HBM saturation, while the unguarded kernel runs ahead, waits on its tile
// loads and then bursts.  Plans with fewer tiles are bound by the step latency and take the
// unguarded kernel (511^2 x 1024: 2.1 vs 2.6 ms per launch).
template <int N, int PP, bool UNI = true, bool GUARD = false>
__global__ void __launch_bounds__(TriTmaCfg<N, PP>::kThreads, 1)
    heat_tridiag_tma_kernel(const __grid_constant__ CUtensorMap map, int64_t inner, int64_t ntc,
                            int64_t l0, const double* __restrict__ lam_col,
                            const double* __restrict__ w_col, double dd, double ds, double cd,
                            double cs, double md, double mo, double ad, double ao,
                            double* __restrict__ carry, const double* __restrict__ d_diag,
                            const double* __restrict__ d_sup, const double* __restrict__ c_diag,
                            const double* __restrict__ c_sup) {
  using C = TriTmaCfg<N, PP>;
  constexpr int R = C::R, T = C::T, n = C::n, W = C::W, LW = C::LW, CW = C::CW;
  extern __shared__ __align__(1024) unsigned char tmraw[];
  if ((static_cast<unsigned>(__cvta_generic_to_shared(tmraw)) & 1023u) != 0u) __trap();
  unsigned char* bout = tmraw + 2 * C::kBufBytes;
  double2* xch = reinterpret_cast<double2*>(tmraw + C::kXchOff);  // [P][8]
  uint64_t* bars = reinterpret_cast<uint64_t*>(tmraw + C::kBarOff);
  uint64_t* full = bars;       // [2] tile landed (TMA transaction bytes)
  uint64_t* empty = bars + 2;  // [2] every warp has read the tile
  uint64_t* ofree = bars + 4;  // the previous store has read the output buffer
  const int tid = threadIdx.x;
  const int f = tid / T, t = tid % T;
  const int sl = t & (W - 1);
  const int bar = 1 + f;
  const int i0 = static_cast<int>(blockIdx.x) * C::G;
  const int64_t ca = i0 + 2 * f;
  const int row0 = R * t;
  const int cnt = n - row0 < 0 ? 0 : (n - row0 > R ? R : n - row0);  // real rows of this chunk
  // Lanes t < TF hold R real rows, lane TF the TAIL = n mod R last ones (then phantom rows),
  // later lanes only phantom rows.  The sweeps below run unguarded over all R rows: phantom
  // rows have zero right-hand sides (zero-filled tile rows, zero z) and their outputs are
  // multiplied by a zero gamma, so they stay exact zeros; the three places where the tail
  // lane's phantom rows would leak into real rows are patched at compile-time positions.
  constexpr int TF = n / R, TAIL = n % R;
  const bool tail_lane = t == TF;
  double2* xp = xch + f * 8;
  // byte offset of this pair's 16-byte chunk in row r of a tile buffer (TMA swizzle)
  const int cbase = (f / C::CPB) * (C::kRows * CW), cc = f % C::CPB;
  auto off = [&](int r) {
    const int sw = CW == 64 ? ((r >> 1) & 3) : (r & 7);
    return cbase + r * CW + ((cc ^ sw) << 4);
  };

  // per-column constants (.x / .y: the pair's two columns)
  double2 q, gam, gamA, gamB, sa, sb, qc, gf, gb, qN, inv, pw0, pw1;
  const double2 wc = make_double2(w_col[ca], w_col[ca + 1]);
  const double lam2[2] = {lam_col[ca], lam_col[ca + 1]};
  const int above = row0 < n ? row0 : n;                      // real rows above the chunk
  const int below = n - row0 - R > 0 ? n - row0 - R : 0;      // real rows below it
  auto setup = [&](double dd_, double ds_, double cd_, double cs_) {
    double qq[2], gg[2], s1[2], s2[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const double la = lam2[c];
      const double p = dd_ + la * cd_;
      const double a = p * mo + cd_ * ao, b = p * md + cd_ * ad;
      const double bp = p * (md + 2.0 * mo) + cd_ * (ad + 2.0 * ao);  // b + 2a
      const double bm = p * (md - 2.0 * mo) + cd_ * (ad - 2.0 * ao);  // b - 2a
      const double sq = sqrt(bp * bm);
      qq[c] = -a / (0.5 * (b + sq));
      gg[c] = 1.0 / sq;
      const double pq = ds_ + la * cs_;
      s1[c] = pq * mo + cs_ * ao;
      s2[c] = pq * md + cs_ * ad;
    }
    q = make_double2(qq[0], qq[1]);
    gam = make_double2(gg[0], gg[1]);
    sa = make_double2(s1[0], s1[1]);
    sb = make_double2(s2[0], s2[1]);
    gamA = t <= TF ? gam : make_double2(0.0, 0.0);  // rows k < TAIL of the chunk
    gamB = t < TF ? gam : make_double2(0.0, 0.0);   // rows k >= TAIL
    qc = make_double2(tri_ipow(q.x, cnt), tri_ipow(q.y, cnt));
    gf = make_double2(tri_ipow(q.x, above), tri_ipow(q.y, above));
    gb = make_double2(tri_ipow(q.x, below), tri_ipow(q.y, below));
    qN = make_double2(tri_ipow(q.x, N), tri_ipow(q.y, N));
    inv = make_double2(1.0 / (1.0 - qN.x * qN.x), 1.0 / (1.0 - qN.y * qN.y));
    constexpr int lo_rows = 32 * R < n ? 32 * R : n;  // real rows of chunks 0..31
    pw0 = make_double2(tri_ipow(q.x, lo_rows), tri_ipow(q.y, lo_rows));
    pw1 = make_double2(tri_ipow(q.x, n - lo_rows), tri_ipow(q.y, n - lo_rows));
  };
  if constexpr (UNI) setup(dd, ds, cd, cs);

  // zero the tile buffers once: rows the TMA boxes never write stay zero; barriers
  for (int e = tid; e < 3 * C::kBufBytes / 16; e += C::kThreads)
    reinterpret_cast<double2*>(tmraw)[e] = make_double2(0.0, 0.0);
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], C::kThreads / 32);
    mbar_init(&empty[1], C::kThreads / 32);
    mbar_init(ofree, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // zeros before the TMA writes
  __syncthreads();

  auto issue_load = [&](int64_t j, int s) {  // one thread
    mbar_arrive_expect_tx(&full[s], C::kTxBytes);
#pragma unroll
    for (int cb = 0; cb < C::NCB; ++cb)
#pragma unroll
      for (int rb = 0; rb < C::NRB; ++rb)
        tma_load_3d(tmraw + s * C::kBufBytes + cb * (C::kRows * CW) + rb * (C::BR * CW), &map,
                    i0 + cb * (CW / 8), rb * C::BR, static_cast<int>(j), &full[s]);
  };
  // The two input buffers bound the load distance to under two steps, less than the DRAM
  // latency under load once a step is short: tiles kPfDist slices ahead are pulled into L2 by
  // TMA prefetches (no shared memory, no barrier), so the loads proper hit L2.
  constexpr int kPfDist = STKG_TRI_PF;
  auto issue_prefetch = [&](int64_t j) {  // one thread
#pragma unroll
    for (int cb = 0; cb < C::NCB; ++cb)
#pragma unroll
      for (int rb = 0; rb < C::NRB; ++rb)
        tma_prefetch_3d(&map, i0 + cb * (CW / 8), rb * C::BR, static_cast<int>(j));
  };
  if (tid == 0) {
    if (ntc > 0) issue_load(0, 0);
    if (ntc > 1) issue_load(1, 1);
    for (int64_t j = 2; j < kPfDist && j < ntc; ++j) issue_prefetch(j);
  }

  // z_{l0-1}: this thread's rows, the row above its first (zu) and below its last (zn)
  double2 x[R], zn = make_double2(0.0, 0.0), zu = make_double2(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int r = row0 + k;
    x[k] = (l0 > 0 && r < n) ? *reinterpret_cast<const double2*>(carry + int64_t(r) * inner + ca)
                             : make_double2(0.0, 0.0);
  }
  if (l0 > 0) {
    if (row0 > 0 && row0 - 1 < n)
      zu = *reinterpret_cast<const double2*>(carry + int64_t(row0 - 1) * inner + ca);
    if (row0 + R < n) zn = *reinterpret_cast<const double2*>(carry + int64_t(row0 + R) * inner + ca);
  }

  for (int64_t j = 0; j < ntc; ++j) {
    const int s = static_cast<int>(j & 1);
    const unsigned ph = static_cast<unsigned>(j >> 1) & 1u;
    if constexpr (!UNI) {
      const int64_t l = l0 + j;
      setup(__ldg(d_diag + l), l > 0 ? __ldg(d_sup + l - 1) : 0.0, __ldg(c_diag + l),
            l > 0 ? __ldg(c_sup + l - 1) : 0.0);
    }
    if (j > 0) {  // the neighbours' edge rows of z_{l-1}
      zu = shfl_up2(x[R - 1], 1, W);
      zn = shfl_down2(x[0], 1, W);
      if (sl == 0) zu = (T > 32 && t == 32) ? xp[4] : make_double2(0.0, 0.0);
      if (sl == W - 1) zn = (T > 32 && t == 31) ? xp[5] : make_double2(0.0, 0.0);
    }
    mbar_wait(&full[s], ph);
    // right-hand side in place: r_i = w_c g_i - sb z_i - sa (z_{i-1} + z_{i+1})
    {
      const unsigned char* tb = tmraw + s * C::kBufBytes;
      double2 zl = zu;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const double2 g = *reinterpret_cast<const double2*>(tb + off(row0 + k));
        const double2 zc = x[k];
        const double2 zr = k + 1 < R ? x[k + 1] : zn;
        // (the first phantom row of the tail lane must not see the last real row above it)
        if (k == TAIL && tail_lane) zl = make_double2(0.0, 0.0);
        const double ra = fma(sb.x, zc.x, sa.x * (zl.x + zr.x));
        const double rb = fma(sb.y, zc.y, sa.y * (zl.y + zr.y));
        x[k] = (!GUARD || k < cnt) ? make_double2(fma(wc.x, g.x, -ra), fma(wc.y, g.y, -rb))
                                   : make_double2(0.0, 0.0);
        zl = zc;
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[s]);  // this warp's reads of the tile are done

    // zero-start recurrences over the chunk, both directions
    double2 ef = make_double2(0.0, 0.0), eb = make_double2(0.0, 0.0);
    double2 cap = make_double2(0.0, 0.0);  // the causal value after the tail lane's real rows
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (!GUARD || k < cnt) {
        ef.x = fma(q.x, ef.x, x[k].x);
        ef.y = fma(q.y, ef.y, x[k].y);
      }
      if (k == TAIL - 1) cap = ef;
      const int kb = R - 1 - k;
      if (!GUARD || kb < cnt) {
        eb.x = fma(q.x, eb.x, x[kb].x);
        eb.y = fma(q.y, eb.y, x[kb].y);
      }
    }
    if (tail_lane) ef = cap;  // (zero-start values of phantom rows are zero: eb needs no patch)
    if (tid == 0) {
      // every warp has read tile j: its buffer takes slice j + 2
      mbar_wait(&empty[s], ph);
      if (j + 2 < ntc) issue_load(j + 2, s);
      if (kPfDist > 2 && j + kPfDist < ntc) issue_prefetch(j + kPfDist);
    }
    // chunk scans (running products of the chunk multipliers q^cnt), both directions
    double2 wf = qc, wb = qc;
#pragma unroll
    for (int k = 0; k < LW; ++k) {
      const int d = 1 << k;
      const double2 vf = shfl_up2(ef, d, W), uf = shfl_up2(wf, d, W);
      const double2 vb = shfl_down2(eb, d, W), ub = shfl_down2(wb, d, W);
      if (sl >= d) {
        ef.x = fma(wf.x, vf.x, ef.x);
        ef.y = fma(wf.y, vf.y, ef.y);
        wf.x *= uf.x;
        wf.y *= uf.y;
      }
      if (sl + d < W) {
        eb.x = fma(wb.x, vb.x, eb.x);
        eb.y = fma(wb.y, vb.y, eb.y);
        wb.x *= ub.x;
        wb.y *= ub.y;
      }
    }
    double2 flo = make_double2(0.0, 0.0), bhi = make_double2(0.0, 0.0);  // across the warps
    double2 an, b1;  // zero-start totals: A at the last row, B at the first
    if constexpr (T > 32) {
      if (t == 31) xp[0] = ef;
      if (t == 32) xp[1] = eb;
      if (t == 63) xp[2] = ef;
      if (t == 0) xp[3] = eb;
      fft_sync<T>(bar);
      const double2 s0 = xp[0], s1 = xp[1], s2 = xp[2], s3 = xp[3];
      if (t >= 32) {
        flo = s0;
        ef.x = fma(wf.x, s0.x, ef.x);
        ef.y = fma(wf.y, s0.y, ef.y);
      } else {
        bhi = s1;
        eb.x = fma(wb.x, s1.x, eb.x);
        eb.y = fma(wb.y, s1.y, eb.y);
      }
      an = make_double2(fma(pw1.x, s0.x, s2.x), fma(pw1.y, s0.y, s2.y));
      b1 = make_double2(fma(pw0.x, s1.x, s3.x), fma(pw0.y, s1.y, s3.y));
    } else {
      const int base = (tid & 31) & ~(W - 1);
      an = make_double2(__shfl_sync(0xffffffffu, ef.x, base + W - 1),
                        __shfl_sync(0xffffffffu, ef.y, base + W - 1));
      b1 = make_double2(__shfl_sync(0xffffffffu, eb.x, base), __shfl_sync(0xffffffffu, eb.y, base));
    }
    // image start values A_0, B_N and this chunk's carry-ins
    double2 fc = shfl_up2(ef, 1, W), bc = shfl_down2(eb, 1, W);
    if (sl == 0) fc = flo;
    if (sl == W - 1) bc = bhi;
    {
      const double aNx = q.x * an.x, aNy = q.y * an.y;
      const double A0x = (qN.x * aNx - q.x * b1.x) * inv.x, A0y = (qN.y * aNy - q.y * b1.y) * inv.y;
      const double BNx = -fma(qN.x, A0x, aNx), BNy = -fma(qN.y, A0y, aNy);
      fc.x = fma(gf.x, A0x, fc.x);
      fc.y = fma(gf.y, A0y, fc.y);
      bc.x = fma(gb.x, BNx, bc.x);
      bc.y = fma(gb.y, BNy, bc.y);
    }
    // causal sweep: A_i in place of r_i
    {
      double2 a = fc;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (!GUARD || k < cnt) {
          a.x = fma(q.x, a.x, x[k].x);
          a.y = fma(q.y, a.y, x[k].y);
          x[k] = a;
        }
      }
    }
    // anti-causal sweep: z_i = gamma (A_i + q B_{i+1}),  B_i = r_i + q B_{i+1}, r_i = A_i - q A_{i-1}
    {
      double2 bn = bc;
#pragma unroll
      for (int k = R - 1; k >= 0; --k) {
        // (the tail lane's sweep enters its last real row with the carry-in itself)
        if (k == TAIL - 1 && tail_lane) bn = bc;
        if (!GUARD || k < cnt) {
          const double2 ak = x[k];
          const double2 am = k > 0 ? x[k - 1] : fc;
          const double2 gk = k < TAIL ? gamA : gamB;
          // r_k = A_k - q A_{k-1} off the chain: one dependent FMA per row on B
          const double rx = fma(-q.x, am.x, ak.x), ry = fma(-q.y, am.y, ak.y);
          x[k] = make_double2(gk.x * fma(q.x, bn.x, ak.x), gk.y * fma(q.y, bn.y, ak.y));
          bn.x = fma(q.x, bn.x, rx);
          bn.y = fma(q.y, bn.y, ry);
        }
      }
    }
    if (tid == 0) {  // the previous slice's store has read the output buffer (long ago)
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      mbar_arrive(ofree);
    }
    mbar_wait(ofree, static_cast<unsigned>(j) & 1u);
#pragma unroll
    for (int k = 0; k < R; ++k) *reinterpret_cast<double2*>(bout + off(row0 + k)) = x[k];
    if constexpr (T > 32) {
      if (t == 31) xp[4] = x[R - 1];
      if (t == 32) xp[5] = x[0];
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
#pragma unroll
      for (int cb = 0; cb < C::NCB; ++cb)
#pragma unroll
        for (int rb = 0; rb < C::NRB; ++rb)
          tma_store_3d(&map, i0 + cb * (CW / 8), rb * C::BR, static_cast<int>(j),
                       bout + cb * (C::kRows * CW) + rb * (C::BR * CW));
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
  }
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int r = row0 + k;
    if (r < n) *reinterpret_cast<double2*>(carry + int64_t(r) * inner + ca) = x[k];
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

}  // namespace stkg
