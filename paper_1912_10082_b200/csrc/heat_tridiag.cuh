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
// per value instead of two FFTs' worth: the pass becomes an HBM stream.  On a uniform time
// grid T is the same for every step, so its LDL^T pivots 1/w_i are computed once per plan
// (tri_factor_kernel) and held in registers.
//
// One CTA owns G = 2P neighbouring columns of axis 0 (all n_0 rows) and marches through the
// time slices.  T = N/16 threads share a column pair; thread t holds rows 16t .. 16t+15 of
// both columns.  The two triangular solves are first-order linear recurrences along the
// rows, run as a chunked scan: every thread runs its 16 rows with zero carry-in, the chunk
// end values are combined across the T threads by a Kogge-Stone scan whose weights (products
// of the chunks' multipliers) are per-plan constants in registers, and every thread reruns
// its rows from its carry-in.  No division, no transform, z_{l-1} stays in registers.
//
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

}  // namespace stkg
