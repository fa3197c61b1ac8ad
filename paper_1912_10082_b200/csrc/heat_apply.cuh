// K1 of the heat hot path: KronOp::apply / the residual (stk/sylvester.hpp:32-38) as
// matrix-free stencil kernels over the 1D tridiagonal factors -- the x-marching 2D and 3D
// kernels and the generic (1D) kernel.  Included by heat.cu only (internal linkage).
#pragma once

#include "common.cuh"
#include "gemm_f64.cuh"  // cp_async8 / commit / wait
#include "heat_plan.cuh"

namespace {
using namespace stkg;

// ------------------------------------------------------------------------------ K1 --
// out_l = M (d_l U_l + ds_{l-1} U_{l-1}) + A (c_l U_l + cs_{l-1} U_{l-1}),
// M = (x) M_a, A = sum_a A_a (x) M_others (fem2d_matrices, stk/discretize.hpp:81-88).
// One thread per spatial point, looping over time; the stencil values of U_{l-1} stay in
// registers, so U and F are each read once from HBM (16 B/unknown).
struct Tri {  // symmetric tridiagonal 1D factor
  const double* diag;
  const double* off;
  __device__ __forceinline__ double w(int64_t i, int q) const {  // entry (i, i+q), q in -1..1
    return q == 0 ? diag[i] : (q < 0 ? off[i - 1] : off[i]);
  }
};

// Tiles of 256 PT points per CTA (x slowest ... fastest axis last); each of the 256
// threads owns PT consecutive points along the fastest axis, so the per-slice overheads
// (ring wait, barrier, copies, time coefficients) are paid once per PT points and a
// thread's 3-point stencils along the fastest axis share loaded values.  The U tile with a
// 1-wide halo (and the F tile for the residual) is staged in shared memory by cp.async in a
// kStages-deep ring over time slices, so every U and F value crosses HBM once and the
// loads for future slices cover the HBM latency.
// Measured (tools/k1_probe.py): 2 points per thread is 5% faster on cfg3 (2D) and 21% on
// cfg5 (3D) than 1; 4 raises registers past two CTAs per SM and loses; 1D keeps 1 (its
// grids are small and a wider tile idles).
template <int NDIM>
constexpr int apply_pt() { return NDIM == 1 ? 1 : 2; }
template <int NDIM> struct ApplyTile;
template <> struct ApplyTile<1> {
  static constexpr int PT = apply_pt<1>(), BX = 256 * PT, BY = 1, BZ = 1, kStages = 6;
};
template <> struct ApplyTile<2> {
  static constexpr int PT = apply_pt<2>(), BX = 8, BY = 32 * PT, BZ = 1, kStages = 6;
};
template <> struct ApplyTile<3> {
  static constexpr int PT = apply_pt<3>(), BX = 4, BY = 4, BZ = 16 * PT, kStages = 6;
};

template <int NDIM, bool RESIDUAL>
struct ApplySmem {
  using T = ApplyTile<NDIM>;
  static constexpr int HX = T::BX + 2, HY = T::BY + (NDIM >= 2 ? 2 : 0);
  static constexpr int HZ = T::BZ + (NDIM == 3 ? 2 : 0);
  static constexpr int TE = HX * HY * HZ;              // halo tile per slice
  static constexpr int TF = RESIDUAL ? 256 * T::PT : 0;  // F tile per slice
  static constexpr size_t kBytes = size_t(T::kStages) * (TE + TF) * sizeof(double);
};

template <int NDIM, bool RESIDUAL>
__global__ void __launch_bounds__(256) heat_apply_kernel(
    const double* __restrict__ U, const double* __restrict__ F, double* __restrict__ out,
    int64_t n0, int64_t n1, int64_t n2, int64_t nt, Tri m0, Tri m1, Tri m2, Tri a0, Tri a1,
    Tri a2, const double* __restrict__ d_diag, const double* __restrict__ d_sup,
    const double* __restrict__ c_diag, const double* __restrict__ c_sup,
    double* __restrict__ partials) {
  using T = ApplyTile<NDIM>;
  using SM = ApplySmem<NDIM, RESIDUAL>;
  constexpr int kPT = T::PT;
  constexpr int HY = SM::HY, HZ = SM::HZ, TE = SM::TE, TF = SM::TF;
  constexpr int kStages = T::kStages;
  extern __shared__ __align__(16) double asmem[];
  double* su = asmem;                      // [kStages][TE]
  double* sf = asmem + kStages * TE;       // [kStages][TF]

  const int64_t tiles_y = (n1 + T::BY - 1) / T::BY, tiles_z = (n2 + T::BZ - 1) / T::BZ;
  int64_t blk = blockIdx.x;
  const int64_t tz = blk % tiles_z;
  blk /= tiles_z;
  const int64_t ty = blk % tiles_y;
  const int64_t tx = blk / tiles_y;
  const int64_t x0 = tx * T::BX, y0 = ty * T::BY, z0 = tz * T::BZ;
  const int tid = threadIdx.x;
  constexpr int TYT = NDIM == 2 ? T::BY / kPT : (NDIM == 3 ? T::BY : 1);
  constexpr int TZT = NDIM == 3 ? T::BZ / kPT : 1;
  const int lx = tid / (TYT * TZT), ly = (tid / TZT) % TYT, lz = tid % TZT;
  const int64_t ix = x0 + (NDIM == 1 ? kPT * lx : lx);
  const int64_t iy = y0 + (NDIM == 2 ? kPT * ly : ly);
  const int64_t iz = z0 + (NDIM == 3 ? kPT * lz : 0);
  const int64_t nx = n0 * n1 * n2;
  const int64_t nf = NDIM == 1 ? n0 : (NDIM == 2 ? n1 : n2);
  const int64_t ifast = NDIM == 1 ? ix : (NDIM == 2 ? iy : iz);
  const bool row_ok = ix < n0 && iy < n1 && iz < n2;
  const int64_t p0 = (ix * n1 + iy) * n2 + iz;

  constexpr int kPer = (TE + 255) / 256;
  int64_t hoff[kPer];
  uint32_t hok = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int e = tid + 256 * k;
    const int hx = e / (HY * HZ), hy = (e / HZ) % HY, hz = e % HZ;
    const int64_t gx = x0 + hx - 1;
    const int64_t gy = NDIM >= 2 ? y0 + hy - 1 : 0;
    const int64_t gz = NDIM == 3 ? z0 + hz - 1 : 0;
    const bool ok = e < TE && gx >= 0 && gx < n0 && gy >= 0 && gy < n1 && gz >= 0 && gz < n2;
    hoff[k] = ok ? (gx * n1 + gy) * n2 + gz : 0;
    if (ok) hok |= 1u << k;
  }
  int64_t foff[kPT];
  uint32_t fok = 0;
  if constexpr (RESIDUAL) {
#pragma unroll
    for (int k = 0; k < kPT; ++k) {
      const int e = tid + 256 * k;
      const int fx = e / (T::BY * T::BZ), fy = (e / T::BZ) % T::BY, fz = e % T::BZ;
      const int64_t gx = x0 + fx, gy = y0 + fy, gz = z0 + fz;
      const bool ok = gx < n0 && gy < n1 && gz < n2;
      foff[k] = ok ? (gx * n1 + gy) * n2 + gz : 0;
      if (ok) fok |= 1u << k;
    }
  }
  auto load_slice = [&](int stage, int64_t l) {
    const bool lin = l < nt;
    const double* Ul = U + l * nx;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int e = tid + 256 * k;
      if (e < TE) {
        const bool ok = lin && ((hok >> k) & 1u);
        cp_async8(&su[stage * TE + e], ok ? Ul + hoff[k] : U, ok);
      }
    }
    if constexpr (RESIDUAL) {
      const double* Fl = F + l * nx;
#pragma unroll
      for (int k = 0; k < kPT; ++k) {
        const bool ok = lin && ((fok >> k) & 1u);
        cp_async8(&sf[stage * TF + tid + 256 * k], ok ? Fl + foff[k] : F, ok);
      }
    }
  };

  auto wts = [&](const Tri& t, int64_t i, int64_t n, int q, bool valid) {
    return (valid && i + q - 1 >= 0 && i + q - 1 < n) ? t.w(i, q - 1) : 0.0;
  };
  double wmf[kPT][3], waf[kPT][3];
  const Tri& mf = NDIM == 1 ? m0 : (NDIM == 2 ? m1 : m2);
  const Tri& af = NDIM == 1 ? a0 : (NDIM == 2 ? a1 : a2);
#pragma unroll
  for (int p = 0; p < kPT; ++p) {
    const bool v = row_ok && ifast + p < nf;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      wmf[p][q] = wts(mf, ifast + p, nf, q, v);
      waf[p][q] = wts(af, ifast + p, nf, q, v);
    }
  }
  double wmx[3], wax[3], wmy[3], way[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    wmx[q] = NDIM >= 2 ? wts(m0, ix, n0, q, row_ok) : 0.0;
    wax[q] = NDIM >= 2 ? wts(a0, ix, n0, q, row_ok) : 0.0;
    wmy[q] = NDIM == 3 ? wts(m1, iy, n1, q, row_ok) : 0.0;
    way[q] = NDIM == 3 ? wts(a1, iy, n1, q, row_ok) : 0.0;
  }

#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) {
    load_slice(st, st);
    cp_async_commit();
  }
  double rr = 0.0, ff = 0.0;
  double mu_prev[kPT], au_prev[kPT];
#pragma unroll
  for (int p = 0; p < kPT; ++p) mu_prev[p] = au_prev[p] = 0.0;
  const int hbase = NDIM == 1 ? kPT * lx
                              : (NDIM == 2 ? lx * HY + kPT * ly : (lx * HY + ly) * HZ + kPT * lz);
  auto dot3 = [](const double* w, double a, double b, double c) {
    return fma(w[2], c, fma(w[1], b, w[0] * a));
  };
  auto line = [&](const double* r, double (&m)[kPT], double (&a)[kPT]) {
    double v[kPT + 2];
#pragma unroll
    for (int k = 0; k < kPT + 2; ++k) v[k] = r[k];
#pragma unroll
    for (int p = 0; p < kPT; ++p) {
      m[p] = dot3(wmf[p], v[p], v[p + 1], v[p + 2]);
      a[p] = dot3(waf[p], v[p], v[p + 1], v[p + 2]);
    }
  };
  int cur = 0, nxt = kStages - 1;
  for (int64_t l = 0; l < nt; ++l) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    load_slice(nxt, l + kStages - 1);
    cp_async_commit();
    const double* t = su + cur * TE + hbase;
    double mu[kPT], au[kPT];
    if constexpr (NDIM == 1) {
      line(t, mu, au);
    } else if constexpr (NDIM == 2) {
      double mr[3][kPT], ar[3][kPT];
#pragma unroll
      for (int qx = 0; qx < 3; ++qx) line(t + qx * HY, mr[qx], ar[qx]);
#pragma unroll
      for (int p = 0; p < kPT; ++p) {
        mu[p] = dot3(wmx, mr[0][p], mr[1][p], mr[2][p]);
        au[p] = dot3(wax, mr[0][p], mr[1][p], mr[2][p]) + dot3(wmx, ar[0][p], ar[1][p], ar[2][p]);
      }
    } else {
      double my[3][kPT], ay[3][kPT];
#pragma unroll
      for (int qx = 0; qx < 3; ++qx) {
        double mz[3][kPT], az[3][kPT];
#pragma unroll
        for (int qy = 0; qy < 3; ++qy) line(t + (qx * HY + qy) * HZ, mz[qy], az[qy]);
#pragma unroll
        for (int p = 0; p < kPT; ++p) {
          my[qx][p] = dot3(wmy, mz[0][p], mz[1][p], mz[2][p]);
          ay[qx][p] = dot3(way, mz[0][p], mz[1][p], mz[2][p]) + dot3(wmy, az[0][p], az[1][p], az[2][p]);
        }
      }
#pragma unroll
      for (int p = 0; p < kPT; ++p) {
        mu[p] = dot3(wmx, my[0][p], my[1][p], my[2][p]);
        au[p] = dot3(wax, my[0][p], my[1][p], my[2][p]) + dot3(wmx, ay[0][p], ay[1][p], ay[2][p]);
      }
    }
    const double dd = d_diag[l], cd = c_diag[l];
    const double ds = l > 0 ? d_sup[l - 1] : 0.0, cs = l > 0 ? c_sup[l - 1] : 0.0;
#pragma unroll
    for (int p = 0; p < kPT; ++p) {
      double acc = dd * mu[p] + cd * au[p];
      if (l > 0) acc += ds * mu_prev[p] + cs * au_prev[p];
      mu_prev[p] = mu[p];
      au_prev[p] = au[p];
      if (row_ok && ifast + p < nf) {
        if constexpr (RESIDUAL) {
          const int e = NDIM == 1 ? kPT * lx + p
                                  : (NDIM == 2 ? lx * T::BY + kPT * ly + p
                                               : (lx * T::BY + ly) * T::BZ + kPT * lz + p);
          const double f = sf[cur * TF + e];
          const double r = f - acc;
          rr += r * r;
          ff += f * f;
        } else {
          out[l * nx + p0 + p] = acc;
        }
      }
    }
    cur = cur + 1 == kStages ? 0 : cur + 1;
    nxt = nxt + 1 == kStages ? 0 : nxt + 1;
  }
  cp_async_wait<0>();
  if (RESIDUAL) {
    __shared__ double red[8];
    rr = block_sum<256>(rr, red);
    ff = block_sum<256>(ff, red);
    if (threadIdx.x == 0) {
      partials[2 * blockIdx.x] = rr;
      partials[2 * blockIdx.x + 1] = ff;
    }
  }
}

// 2D K1, marching along x.  A thread owns PT = 4 consecutive points along x at one y
// (a warp = 32 consecutive y, coalesced), so the y-direction products of a U row
// (m = M_y u, a = A_y u: 6 FMA) are shared by the up-to-3 points that use that row
// instead of being recomputed per point: (PT + 2) / PT x 6 + 9 FMA per point for M U and
// A U instead of 27 (heat_apply_kernel<2>).  The x weights of the thread's 4 points stay
// in registers as diag[4] / off[5] (the factors are symmetric tridiagonal).  A CTA handles
// a 32 x 32 tile over a chunk of kChunk time slices, first re-deriving M U, A U of the
// slice before its chunk, so the grid has tiles x chunks CTAs (no half-empty last wave).
struct Apply2D {
  static constexpr int PT = 4, SEG = 8, BY = 32, BX = PT * SEG;
  static constexpr int HX = BX + 2, HY = BY + 2, TE = HX * HY, TF = BX * BY;
  static constexpr int kStages = 4, kChunk = 64;
  static constexpr int kPer = (TE + 255) / 256, kPerF = TF / 256;
};
template <bool RESIDUAL>
constexpr size_t apply2d_smem() {
  return size_t(Apply2D::kStages) * (Apply2D::TE + (RESIDUAL ? Apply2D::TF : 0)) * sizeof(double);
}

template <bool RESIDUAL>
__global__ void __launch_bounds__(256, 2) heat_apply2d_kernel(
    const double* __restrict__ U, const double* __restrict__ F, double* __restrict__ out,
    int64_t n0, int64_t n1, int64_t nt, Tri m0, Tri m1, Tri a0, Tri a1,
    const double* __restrict__ d_diag, const double* __restrict__ d_sup,
    const double* __restrict__ c_diag, const double* __restrict__ c_sup,
    double* __restrict__ partials) {
  using A = Apply2D;
  constexpr int PT = A::PT, HY = A::HY, TE = A::TE, TF = A::TF, kStages = A::kStages;
  extern __shared__ __align__(16) double asmem[];
  double* su = asmem;                  // [kStages][TE]
  double* sf = asmem + kStages * TE;   // [kStages][TF]
  const int64_t tiles_y = (n1 + A::BY - 1) / A::BY, tiles_x = (n0 + A::BX - 1) / A::BX;
  const int64_t tile = blockIdx.x % (tiles_x * tiles_y), ck = blockIdx.x / (tiles_x * tiles_y);
  const int64_t x0 = (tile / tiles_y) * A::BX, y0 = (tile % tiles_y) * A::BY;
  const int64_t l_begin = ck * A::kChunk;
  const int64_t l_end = l_begin + A::kChunk < nt ? l_begin + A::kChunk : nt;
  const int64_t l_first = l_begin > 0 ? l_begin - 1 : 0;  // warm-up slice for M U_{l-1}
  const int tid = threadIdx.x, lane = tid & 31, seg = tid >> 5;
  const int64_t iy = y0 + lane, xs = x0 + seg * PT;
  const int64_t nx = n0 * n1;

  int64_t hoff[A::kPer];
  uint32_t hok = 0;
#pragma unroll
  for (int k = 0; k < A::kPer; ++k) {
    const int e = tid + 256 * k;
    const int64_t gx = x0 + e / HY - 1, gy = y0 + e % HY - 1;
    const bool ok = e < TE && gx >= 0 && gx < n0 && gy >= 0 && gy < n1;
    hoff[k] = ok ? gx * n1 + gy : 0;
    if (ok) hok |= 1u << k;
  }
  int64_t foff[A::kPerF];
  uint32_t fok = 0;
  if constexpr (RESIDUAL) {
#pragma unroll
    for (int k = 0; k < A::kPerF; ++k) {
      const int e = tid + 256 * k;
      const int64_t gx = x0 + e / A::BY, gy = y0 + e % A::BY;
      const bool ok = gx < n0 && gy < n1;
      foff[k] = ok ? gx * n1 + gy : 0;
      if (ok) fok |= 1u << k;
    }
  }
  auto load_slice = [&](int stage, int64_t l) {
    const bool lin = l < l_end;
    const double* Ul = U + l * nx;
#pragma unroll
    for (int k = 0; k < A::kPer; ++k) {
      const int e = tid + 256 * k;
      if (e < TE) {
        const bool ok = lin && ((hok >> k) & 1u);
        cp_async8(&su[stage * TE + e], ok ? Ul + hoff[k] : U, ok);
      }
    }
    if constexpr (RESIDUAL) {
      const double* Fl = F + l * nx;
#pragma unroll
      for (int k = 0; k < A::kPerF; ++k) {
        const bool ok = lin && l >= l_begin && ((fok >> k) & 1u);
        cp_async8(&sf[stage * TF + tid + 256 * k], ok ? Fl + foff[k] : F, ok);
      }
    }
  };

  // y weights of this thread's row; x weights of its PT points (symmetric tridiagonals)
  const bool y_ok = iy < n1;
  double wmy[3], way[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int64_t j = iy + q - 1;
    const bool ok = y_ok && j >= 0 && j < n1;
    wmy[q] = ok ? m1.w(iy, q - 1) : 0.0;
    way[q] = ok ? a1.w(iy, q - 1) : 0.0;
  }
  double md[PT], ad[PT], mo[PT + 1], ao[PT + 1];
#pragma unroll
  for (int p = 0; p < PT; ++p) {
    const bool ok = xs + p < n0;
    md[p] = ok ? m0.diag[xs + p] : 0.0;
    ad[p] = ok ? a0.diag[xs + p] : 0.0;
  }
#pragma unroll
  for (int k = 0; k <= PT; ++k) {  // off[xs - 1 + k]: entry (x, x+1) for x = xs - 1 + k
    const int64_t x = xs - 1 + k;
    const bool ok = x >= 0 && x + 1 < n0;
    mo[k] = ok ? m0.off[x] : 0.0;
    ao[k] = ok ? a0.off[x] : 0.0;
  }

#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) {
    load_slice(st, l_first + st);
    cp_async_commit();
  }
  double rr = 0.0, ff = 0.0;
  double mu_prev[PT], au_prev[PT];
#pragma unroll
  for (int p = 0; p < PT; ++p) mu_prev[p] = au_prev[p] = 0.0;
  const int hbase = seg * PT * HY + lane;
  int cur = 0, nxt = kStages - 1;
  for (int64_t l = l_first; l < l_end; ++l) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    load_slice(nxt, l + kStages - 1);
    cp_async_commit();
    const double* t = su + cur * TE + hbase;
    double mr[PT + 2], ar[PT + 2];
#pragma unroll
    for (int r = 0; r < PT + 2; ++r) {
      const double v0 = t[r * HY], v1 = t[r * HY + 1], v2 = t[r * HY + 2];
      mr[r] = fma(wmy[2], v2, fma(wmy[1], v1, wmy[0] * v0));
      ar[r] = fma(way[2], v2, fma(way[1], v1, way[0] * v0));
    }
    double mu[PT], au[PT];
#pragma unroll
    for (int p = 0; p < PT; ++p) {
      mu[p] = fma(mo[p + 1], mr[p + 2], fma(md[p], mr[p + 1], mo[p] * mr[p]));
      au[p] = fma(ao[p + 1], mr[p + 2], fma(ad[p], mr[p + 1], ao[p] * mr[p])) +
              fma(mo[p + 1], ar[p + 2], fma(md[p], ar[p + 1], mo[p] * ar[p]));
    }
    if (l >= l_begin) {
      const double dd = d_diag[l], cd = c_diag[l];
      const double ds = l > 0 ? d_sup[l - 1] : 0.0, cs = l > 0 ? c_sup[l - 1] : 0.0;
#pragma unroll
      for (int p = 0; p < PT; ++p) {
        double acc = dd * mu[p] + cd * au[p];
        if (l > 0) acc += ds * mu_prev[p] + cs * au_prev[p];
        if (y_ok && xs + p < n0) {
          if constexpr (RESIDUAL) {
            const double f = sf[cur * TF + (seg * PT + p) * A::BY + lane];
            const double r = f - acc;
            rr += r * r;
            ff += f * f;
          } else {
            out[l * nx + (xs + p) * n1 + iy] = acc;
          }
        }
      }
    }
#pragma unroll
    for (int p = 0; p < PT; ++p) {
      mu_prev[p] = mu[p];
      au_prev[p] = au[p];
    }
    cur = cur + 1 == kStages ? 0 : cur + 1;
    nxt = nxt + 1 == kStages ? 0 : nxt + 1;
  }
  cp_async_wait<0>();
  if (RESIDUAL) {
    __shared__ double red[8];
    rr = block_sum<256>(rr, red);
    ff = block_sum<256>(ff, red);
    if (threadIdx.x == 0) {
      partials[2 * blockIdx.x] = rr;
      partials[2 * blockIdx.x + 1] = ff;
    }
  }
}

// 3D K1, marching along x (the 2D kernel's structure one dimension up).  A thread owns
// PT = 4 consecutive points along x at one (y, z) (a warp = 32 consecutive z, one y per
// warp): the (y, z)-plane products of each of its 6 x-rows -- M_yz u = (M_y (x) M_z) u and
// A_yz u = (A_y (x) M_z + M_y (x) A_z) u from the 3 x 3 neighbourhood, 27 FMA -- are formed
// once and combined along x with the thread's x weights: (6/4) 27 + 9 = 49.5 FMA and
// 13.5 shared loads per point instead of about 90 and 18.
struct Apply3D {
  static constexpr int PT = 4, BZ = 32, BY = 8, BX = PT;
  static constexpr int HX = BX + 2, HY = BY + 2, HZ = BZ + 2, TE = HX * HY * HZ;
  static constexpr int TF = BX * BY * BZ;
  static constexpr int kStages = 3, kChunk = 64;
  static constexpr int kPer = (TE + 255) / 256, kPerF = TF / 256;
};
template <bool RESIDUAL>
constexpr size_t apply3d_smem() {
  return size_t(Apply3D::kStages) * (Apply3D::TE + (RESIDUAL ? Apply3D::TF : 0)) * sizeof(double);
}

template <bool RESIDUAL>
__global__ void __launch_bounds__(256, 2) heat_apply3d_kernel(
    const double* __restrict__ U, const double* __restrict__ F, double* __restrict__ out,
    int64_t n0, int64_t n1, int64_t n2, int64_t nt, Tri m0, Tri m1, Tri m2, Tri a0, Tri a1,
    Tri a2, const double* __restrict__ d_diag, const double* __restrict__ d_sup,
    const double* __restrict__ c_diag, const double* __restrict__ c_sup,
    double* __restrict__ partials) {
  using A = Apply3D;
  constexpr int PT = A::PT, HY = A::HY, HZ = A::HZ, TE = A::TE, TF = A::TF;
  constexpr int kStages = A::kStages;
  extern __shared__ __align__(16) double asmem[];
  double* su = asmem;                  // [kStages][TE]
  double* sf = asmem + kStages * TE;   // [kStages][TF]
  const int64_t tz_n = (n2 + A::BZ - 1) / A::BZ, ty_n = (n1 + A::BY - 1) / A::BY;
  const int64_t tx_n = (n0 + A::BX - 1) / A::BX, ntile = tx_n * ty_n * tz_n;
  int64_t tile = blockIdx.x % ntile;
  const int64_t ck = blockIdx.x / ntile;
  const int64_t z0 = (tile % tz_n) * A::BZ;
  tile /= tz_n;
  const int64_t y0 = (tile % ty_n) * A::BY, x0 = (tile / ty_n) * A::BX;
  const int64_t l_begin = ck * A::kChunk;
  const int64_t l_end = l_begin + A::kChunk < nt ? l_begin + A::kChunk : nt;
  const int64_t l_first = l_begin > 0 ? l_begin - 1 : 0;
  const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
  const int64_t iz = z0 + lane, iy = y0 + wy;
  const int64_t nx = n0 * n1 * n2;

  int64_t hoff[A::kPer];
  uint32_t hok = 0;
#pragma unroll
  for (int k = 0; k < A::kPer; ++k) {
    const int e = tid + 256 * k;
    const int hx = e / (HY * HZ), hy = (e / HZ) % HY, hz = e % HZ;
    const int64_t gx = x0 + hx - 1, gy = y0 + hy - 1, gz = z0 + hz - 1;
    const bool ok = e < TE && gx >= 0 && gx < n0 && gy >= 0 && gy < n1 && gz >= 0 && gz < n2;
    hoff[k] = ok ? (gx * n1 + gy) * n2 + gz : 0;
    if (ok) hok |= 1u << k;
  }
  int64_t foff[A::kPerF];
  uint32_t fok = 0;
  if constexpr (RESIDUAL) {
#pragma unroll
    for (int k = 0; k < A::kPerF; ++k) {
      const int e = tid + 256 * k;  // e = (fx * BY + fy) * BZ + fz
      const int64_t gx = x0 + e / (A::BY * A::BZ), gy = y0 + (e / A::BZ) % A::BY,
                    gz = z0 + e % A::BZ;
      const bool ok = gx < n0 && gy < n1 && gz < n2;
      foff[k] = ok ? (gx * n1 + gy) * n2 + gz : 0;
      if (ok) fok |= 1u << k;
    }
  }
  auto load_slice = [&](int stage, int64_t l) {
    const bool lin = l < l_end;
    const double* Ul = U + l * nx;
#pragma unroll
    for (int k = 0; k < A::kPer; ++k) {
      const int e = tid + 256 * k;
      if (e < TE) {
        const bool ok = lin && ((hok >> k) & 1u);
        cp_async8(&su[stage * TE + e], ok ? Ul + hoff[k] : U, ok);
      }
    }
    if constexpr (RESIDUAL) {
      const double* Fl = F + l * nx;
#pragma unroll
      for (int k = 0; k < A::kPerF; ++k) {
        const bool ok = lin && l >= l_begin && ((fok >> k) & 1u);
        cp_async8(&sf[stage * TF + tid + 256 * k], ok ? Fl + foff[k] : F, ok);
      }
    }
  };

  const bool yz_ok = iy < n1 && iz < n2;
  double wmz[3], waz[3], wmy[3], way[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int64_t jz = iz + q - 1, jy = iy + q - 1;
    const bool okz = yz_ok && jz >= 0 && jz < n2, oky = yz_ok && jy >= 0 && jy < n1;
    wmz[q] = okz ? m2.w(iz, q - 1) : 0.0;
    waz[q] = okz ? a2.w(iz, q - 1) : 0.0;
    wmy[q] = oky ? m1.w(iy, q - 1) : 0.0;
    way[q] = oky ? a1.w(iy, q - 1) : 0.0;
  }
  double md[PT], ad[PT], mo[PT + 1], ao[PT + 1];
#pragma unroll
  for (int p = 0; p < PT; ++p) {
    const bool ok = x0 + p < n0;
    md[p] = ok ? m0.diag[x0 + p] : 0.0;
    ad[p] = ok ? a0.diag[x0 + p] : 0.0;
  }
#pragma unroll
  for (int k = 0; k <= PT; ++k) {
    const int64_t x = x0 - 1 + k;
    const bool ok = x >= 0 && x + 1 < n0;
    mo[k] = ok ? m0.off[x] : 0.0;
    ao[k] = ok ? a0.off[x] : 0.0;
  }

#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) {
    load_slice(st, l_first + st);
    cp_async_commit();
  }
  double rr = 0.0, ff = 0.0;
  double mu_prev[PT], au_prev[PT];
#pragma unroll
  for (int p = 0; p < PT; ++p) mu_prev[p] = au_prev[p] = 0.0;
  const int hbase = wy * HZ + lane;
  int cur = 0, nxt = kStages - 1;
  for (int64_t l = l_first; l < l_end; ++l) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    load_slice(nxt, l + kStages - 1);
    cp_async_commit();
    const double* t = su + cur * TE + hbase;
    double mr[PT + 2], ar[PT + 2];
#pragma unroll
    for (int r = 0; r < PT + 2; ++r) {
      double zm[3], za[3];
#pragma unroll
      for (int qy = 0; qy < 3; ++qy) {
        const double* row = t + (r * HY + qy) * HZ;
        const double v0 = row[0], v1 = row[1], v2 = row[2];
        zm[qy] = fma(wmz[2], v2, fma(wmz[1], v1, wmz[0] * v0));
        za[qy] = fma(waz[2], v2, fma(waz[1], v1, waz[0] * v0));
      }
      mr[r] = fma(wmy[2], zm[2], fma(wmy[1], zm[1], wmy[0] * zm[0]));
      ar[r] = fma(way[2], zm[2], fma(way[1], zm[1], way[0] * zm[0])) +
              fma(wmy[2], za[2], fma(wmy[1], za[1], wmy[0] * za[0]));
    }
    double mu[PT], au[PT];
#pragma unroll
    for (int p = 0; p < PT; ++p) {
      mu[p] = fma(mo[p + 1], mr[p + 2], fma(md[p], mr[p + 1], mo[p] * mr[p]));
      au[p] = fma(ao[p + 1], mr[p + 2], fma(ad[p], mr[p + 1], ao[p] * mr[p])) +
              fma(mo[p + 1], ar[p + 2], fma(md[p], ar[p + 1], mo[p] * ar[p]));
    }
    if (l >= l_begin) {
      const double dd = d_diag[l], cd = c_diag[l];
      const double ds = l > 0 ? d_sup[l - 1] : 0.0, cs = l > 0 ? c_sup[l - 1] : 0.0;
#pragma unroll
      for (int p = 0; p < PT; ++p) {
        double acc = dd * mu[p] + cd * au[p];
        if (l > 0) acc += ds * mu_prev[p] + cs * au_prev[p];
        if (yz_ok && x0 + p < n0) {
          if constexpr (RESIDUAL) {
            const double f = sf[cur * TF + (p * A::BY + wy) * A::BZ + lane];
            const double r = f - acc;
            rr += r * r;
            ff += f * f;
          } else {
            out[l * nx + ((x0 + p) * n1 + iy) * n2 + iz] = acc;
          }
        }
      }
    }
#pragma unroll
    for (int p = 0; p < PT; ++p) {
      mu_prev[p] = mu[p];
      au_prev[p] = au[p];
    }
    cur = cur + 1 == kStages ? 0 : cur + 1;
    nxt = nxt + 1 == kStages ? 0 : nxt + 1;
  }
  cp_async_wait<0>();
  if (RESIDUAL) {
    __shared__ double red[8];
    rr = block_sum<256>(rr, red);
    ff = block_sum<256>(ff, red);
    if (threadIdx.x == 0) {
      partials[2 * blockIdx.x] = rr;
      partials[2 * blockIdx.x + 1] = ff;
    }
  }
}

}  // namespace
