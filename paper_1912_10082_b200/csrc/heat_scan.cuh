// K3 of the heat hot path: the per-mode temporal recurrence of solve_projected_heat_with
// (stk/sylvester.hpp:128-140) -- one chain per mode (heat_scan_kernel), the
// parallel-in-time chunked form for plans with few modes, the factored-load form, and the
// plan-time singularity check.  Included by heat.cu only (internal linkage).
#pragma once

#include "common.cuh"
#include "heat_plan.cuh"

namespace {
using namespace stkg;

// ------------------------------------------------------------------------------ K3 --
// One thread per mode i: y_j = (g~_j - (d_sup[j-1] + lam_i c_sup[j-1]) y_{j-1}) /
// (d_diag[j] + lam_i c_diag[j]) -- the forward substitution of stk/sylvester.hpp:131-139,
// with lam_i = lam_x[ix] + lam_y[iy] (+ lam_z[iz]).  Loads of g~ are independent of the
// carried y, so the unrolled loop keeps many of them in flight (HBM-bound, 16 B/unknown).
// Optional per-mode output weight w_i = prod_a w_a[i_a] (P1_DST backend: 1/(mu_x mu_y ..)).
struct ModeWeight {
  const double* w0;
  const double* w1;
  const double* w2;
  int64_t n1, n2;
  int ndim;
  __device__ __forceinline__ double operator()(int64_t i) const {
    if (!w0) return 1.0;
    if (ndim == 1) return w0[i];
    if (ndim == 2) return w0[i / n1] * w1[i % n1];
    const int64_t iz = i % n2, r = i / n2;
    return w0[r / n1] * w1[r % n1] * w2[iz];
  }
};

__global__ void __launch_bounds__(256) heat_scan_kernel(
    double* __restrict__ Y, int64_t nx, int64_t ntc, int64_t l0, ModeLambda lam, ModeWeight wgt,
    const double* __restrict__ d_diag, const double* __restrict__ d_sup,
    const double* __restrict__ c_diag, const double* __restrict__ c_sup,
    double* __restrict__ carry) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nx) return;
  const double li = lam(i);
  const double wi = wgt(i);  // 1 in the dense backend
  double y = l0 > 0 ? carry[i] : 0.0;
  double* col = Y + i;
#ifndef STKG_SCAN_U
#define STKG_SCAN_U 8
#endif
  constexpr int U = STKG_SCAN_U;
  int64_t j = 0;
  // software-pipelined: the next block's U loads are in flight while this block's
  // dependent recurrence runs
  double g[U];
  if (ntc >= U) {
#pragma unroll
    for (int u = 0; u < U; ++u) g[u] = __ldcs(col + u * nx);
  }
  for (; j + U <= ntc; j += U) {
    double gn[U];
    const bool more = j + 2 * U <= ntc;
#pragma unroll
    for (int u = 0; u < U; ++u) gn[u] = more ? __ldcs(col + (j + U + u) * nx) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t l = l0 + j + u;
      const double piv = d_diag[l] + li * c_diag[l];
      double rhs = g[u];
      if (l > 0) rhs -= (d_sup[l - 1] + li * c_sup[l - 1]) * y;
      y = rhs / piv;
      __stcs(col + (j + u) * nx, wi * y);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) g[u] = gn[u];
  }
  for (; j < ntc; ++j) {
    const int64_t l = l0 + j;
    const double piv = d_diag[l] + li * c_diag[l];
    double rhs = col[j * nx];
    if (l > 0) rhs -= (d_sup[l - 1] + li * c_sup[l - 1]) * y;
    y = rhs / piv;
    col[j * nx] = wi * y;
  }
  carry[i] = y;
}

// Parallel-in-time K3 for plans with few modes (the north_star's "parallel scans batched
// over modes"): with n_x <= 2^17 one thread per mode leaves most of the GPU idle and the
// solve is bound by the n_t-step dependency chain.  A CTA of 32 x 32 threads takes 32
// consecutive modes (lane = mode, coalesced) and cuts time into 32 chunks (warp w = chunk
// w).  Phase 1: every thread composes its chunk's affine steps y -> a y + g/piv into
// (A, B); phase 2: warp 0 chains the 32 composites into each chunk's carry-in; phase 3:
// every thread reruns its chunk from its carry-in with the reference's step
// y = (g - sub y) / piv.  The dependency chain drops from n_t to about 2 n_t/32 + 32 steps;
// the carries differ from the sequential ones in rounding only (P1_DST plans, whose
// host-buffer path is not bitwise-equal to the device path anyway), and g is read twice.
// LREG > 0: chunks of at most LREG steps keep their g in registers between phases 1 and
// 3 (g read once, 16 B/unknown as in heat_scan_kernel); LREG = 0: g is re-read in phase 3.
constexpr int64_t kChunkedScanMaxModes = int64_t(1) << 17;
template <int LREG>
__global__ void __launch_bounds__(1024) heat_scan_chunked_kernel(
    double* __restrict__ Y, int64_t nx, int64_t ntc, int64_t l0, ModeLambda lam, ModeWeight wgt,
    const double* __restrict__ d_diag, const double* __restrict__ d_sup,
    const double* __restrict__ c_diag, const double* __restrict__ c_sup,
    double* __restrict__ carry) {
  __shared__ double sA[32][33], sB[32][33];  // [chunk][mode]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i = int64_t(blockIdx.x) * 32 + lane;
  const bool ok = i < nx;
  const int64_t L = (ntc + 31) / 32, lb = w * L, le = lb + L < ntc ? lb + L : ntc;
  const double li = ok ? lam(i) : 0.0, wi = ok ? wgt(i) : 0.0;
  double A = 1.0, B = 0.0;
  double gr[LREG > 0 ? LREG : 1];
  // LREG > 0 (uniform grids): y = (g - sub y) / piv with the mode's constant piv, sub
  const double upiv = d_diag[0] + li * c_diag[0];
  const double usub = ntc + l0 > 1 ? d_sup[0] + li * c_sup[0] : 0.0;
  const double urp = LREG > 0 ? 1.0 / upiv : 0.0, ua = -usub * urp;
  if constexpr (LREG > 0) {
#pragma unroll
    for (int k = 0; k < LREG; ++k) gr[k] = (ok && lb + k < le) ? __ldcs(Y + (lb + k) * nx + i) : 0.0;
  }
  if (ok) {
    if constexpr (LREG > 0) {  // uniform time grid: one pivot and coupling per mode
#pragma unroll
      for (int k = 0; k < LREG; ++k) {
        if (lb + k < le) {
          const double a = l0 + lb + k > 0 ? ua : 0.0;
          A *= a;
          B = fma(a, B, gr[k] * urp);
        }
      }
    } else {
      for (int64_t l = lb; l < le; ++l) {
        const int64_t gl = l0 + l;
        const double piv = d_diag[gl] + li * c_diag[gl];
        const double sub = gl > 0 ? d_sup[gl - 1] + li * c_sup[gl - 1] : 0.0;
        const double a = -sub / piv;
        A *= a;
        B = fma(a, B, __ldcs(Y + l * nx + i) / piv);
      }
    }
  }
  sA[w][lane] = A;
  sB[w][lane] = B;
  __syncthreads();
  if (w == 0) {
    double c = (ok && l0 > 0) ? carry[i] : 0.0;
    for (int k = 0; k < 32; ++k) {
      const double a = sA[k][lane], b = sB[k][lane];
      sA[k][lane] = c;  // carry-in y_{lb - 1} of chunk k
      c = fma(a, c, b);
    }
  }
  __syncthreads();
  double y = sA[w][lane];
  if (ok && lb < le) {
    if constexpr (LREG > 0) {
#pragma unroll
      for (int k = 0; k < LREG; ++k) {
        if (lb + k < le) {
          double rhs = gr[k];
          if (l0 + lb + k > 0) rhs -= usub * y;
          y = rhs * urp;
          __stcs(Y + (lb + k) * nx + i, wi * y);
        }
      }
    } else {
      for (int64_t l = lb; l < le; ++l) {
        const int64_t gl = l0 + l;
        const double piv = d_diag[gl] + li * c_diag[gl];
        double rhs = Y[l * nx + i];
        if (gl > 0) rhs -= (d_sup[gl - 1] + li * c_sup[gl - 1]) * y;
        y = rhs / piv;
        __stcs(Y + l * nx + i, wi * y);
      }
    }
    if (le == ntc) carry[i] = y;
  }
}

// Which K3 kernel a scan over nm modes and ntc steps uses: 0 = heat_scan_kernel (one
// chain per mode), 1 = chunked with g in registers (ntc <= 32 * 16), 2 = chunked with g
// re-read (only for very few modes, where the chain latency dwarfs the second read).
// Measured (cfg1 1D 255 x 256): 53.5 -> 14.6 us with the re-read form; the re-read form
// lost at cfg2 (65,280 modes x 512: 215 -> 267 us, it moves 24 B/unknown).
int scan_variant(const stkg_heat& h, int64_t nm, int64_t ntc) {
  static const bool on = !(std::getenv("STKG_SCAN_CHUNKED") && std::getenv("STKG_SCAN_CHUNKED")[0] == '0');
  if (!on || h.transform != STKG_TRANSFORM_P1_DST || nm > kChunkedScanMaxModes) return 0;
  if (h.uniform_time && ntc <= 32 * 16) return 1;
  return nm <= 8192 ? 2 : 0;
}

template <class LAM, class WGT>
void launch_scan(const stkg_heat& h, double* Y, int64_t nm, int64_t ntc, int64_t l0, LAM lam,
                 WGT wgt) {
  const int v = scan_variant(h, nm, ntc);
  if (v == 1)
    heat_scan_chunked_kernel<16><<<static_cast<unsigned>(ceil_div(nm, 32)), 1024, 0, h.stream>>>(
        Y, nm, ntc, l0, lam, wgt, h.d_diag.p, h.d_sup.p, h.c_diag.p, h.c_sup.p, h.carry.p);
  else if (v == 2)
    heat_scan_chunked_kernel<0><<<static_cast<unsigned>(ceil_div(nm, 32)), 1024, 0, h.stream>>>(
        Y, nm, ntc, l0, lam, wgt, h.d_diag.p, h.d_sup.p, h.c_diag.p, h.c_sup.p, h.carry.p);
  else
    heat_scan_kernel<<<static_cast<unsigned>(ceil_div(nm, 256)), 256, 0, h.stream>>>(
        Y, nm, ntc, l0, lam, wgt, h.d_diag.p, h.d_sup.p, h.c_diag.p, h.c_sup.p, h.carry.p);
  STKG_CUDA_CHECK(cudaGetLastError());
}

// Factored load F = L R^T: the transformed load is never stored;
// g~_j[i] = sum_r Lt[i, r] R[j, r] is formed in registers (Lt = X^T L, n_x x rank), and the
// recurrence writes Y~ (n_x x n_t) -- 8 B/unknown of HBM traffic instead of 16.
constexpr int kMaxFactorRank = 16;
//
// UNI (uniform time grid: every d_j, c_j, d^s_j, c^s_j equal): the pivot and coupling of a
// mode are the same at every step, so the step is y = (g - b y) * (1 / piv) with the
// reciprocal formed once per mode.  Without a transformed load to stream this kernel is
// bound by the per-step FP64 division (a ~25-instruction Newton sequence), not by its
// 8 B/unknown of stores; the reciprocal differs from the reference's division by at most
// an ulp per step.
// RP: the rank rounded up to 2/4/8/16; Rt holds R transposed and zero-padded, Rt[l RP + r]
// (factor_transpose_kernel), so a step's RP coefficients are RP/2 broadcast 16-byte loads
// (indexing R[r nt + l] under a runtime rank cost ~190 instructions per warp and step).
template <bool UNI, int RP>
__global__ void __launch_bounds__(256) heat_scan_factored_kernel(
    const double* __restrict__ Lt, const double* __restrict__ Rt, int rank, double* __restrict__ Y,
    int64_t nx, int64_t nt, ModeLambda lam, ModeWeight wgt, const double* __restrict__ d_diag,
    const double* __restrict__ d_sup, const double* __restrict__ c_diag,
    const double* __restrict__ c_sup, int64_t pitch, int64_t nl) {
  // pitch > 0: Y in the padded layout (nx counts padded modes; Lt stays unpadded with
  // nx / pitch * nl rows; pad lanes get a zero load)
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nx) return;
  const double li = lam(i);
  const double wi = wgt(i);
  int64_t iu = i, nxu = nx;
  bool pad = false;
  if (pitch > 0) {
    const int64_t q = i / pitch, rr = i - q * pitch;
    iu = q * nl + rr;
    nxu = nx / pitch * nl;
    pad = rr >= nl;
  }
  double lt[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r)
    lt[r] = (r < rank && !pad) ? Lt[int64_t(r) * nxu + iu] : 0.0;
  auto load_g = [&](int64_t l) {
    const double2* rl = reinterpret_cast<const double2*>(Rt + l * RP);
    double g = 0.0;
#pragma unroll
    for (int k = 0; k < RP / 2; ++k) {
      const double2 v = __ldg(rl + k);
      g = fma(lt[2 * k], v.x, g);
      g = fma(lt[2 * k + 1], v.y, g);
    }
    return g;
  };
  double y = 0.0;
  if constexpr (UNI) {
    const double rpiv = 1.0 / (d_diag[0] + li * c_diag[0]);
    const double b = nt > 1 ? d_sup[0] + li * c_sup[0] : 0.0;
    for (int64_t l = 0; l < nt; ++l) {
      const double g = load_g(l);
      y = fma(-b, y, g) * rpiv;  // y_{-1} = 0
      __stcs(Y + l * nx + i, wi * y);
    }
  } else {
    for (int64_t l = 0; l < nt; ++l) {
      double g = load_g(l);
      const double piv = d_diag[l] + li * c_diag[l];
      if (l > 0) g -= (d_sup[l - 1] + li * c_sup[l - 1]) * y;
      y = g / piv;
      __stcs(Y + l * nx + i, wi * y);
    }
  }
}

using FactoredScanFn = void (*)(const double*, const double*, int, double*, int64_t, int64_t,
                               ModeLambda, ModeWeight, const double*, const double*,
                               const double*, const double*, int64_t, int64_t);
int factor_rp(int64_t rank) { return rank <= 2 ? 2 : rank <= 4 ? 4 : rank <= 8 ? 8 : 16; }
template <bool UNI>
FactoredScanFn factored_fn(int rp) {
  switch (rp) {
    case 2: return heat_scan_factored_kernel<UNI, 2>;
    case 4: return heat_scan_factored_kernel<UNI, 4>;
    case 8: return heat_scan_factored_kernel<UNI, 8>;
    default: return heat_scan_factored_kernel<UNI, 16>;
  }
}
FactoredScanFn launch_factored(bool uniform, int rp) {
  static const bool on = !(std::getenv("STKG_SCAN_RECIP") && std::getenv("STKG_SCAN_RECIP")[0] == '0');
  return uniform && on ? factored_fn<true>(rp) : factored_fn<false>(rp);
}

// Rt[l rp + r] = R[r nt + l] for r < rank, 0 for rank <= r < rp.
__global__ void factor_transpose_kernel(const double* __restrict__ R, int64_t rank, int64_t nt,
                                        int rp, double* __restrict__ Rt) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= nt * rp) return;
  const int64_t l = e / rp, r = e % rp;
  Rt[e] = r < rank ? R[r * nt + l] : 0.0;
}

// Singularity check of stk/sylvester.hpp:133-135, done once per plan: min over modes and
// steps of |d_j + lambda_i c_j|.  Writes the first offending (i, j) it finds.
__global__ void heat_pivot_check_kernel(int64_t nx, int64_t nt, ModeLambda lam,
                                        const double* d_diag, const double* c_diag,
                                        unsigned long long* bad) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nx) return;
  const double li = lam(i);
  for (int64_t l = 0; l < nt; ++l) {
    const double piv = d_diag[l] + li * c_diag[l];
    if (fabs(piv) < 1e-300) {
      atomicMin(bad, (unsigned long long)(l * nx + i));
      return;
    }
  }
}

}  // namespace
