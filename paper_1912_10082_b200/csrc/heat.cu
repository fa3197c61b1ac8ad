// Heat hot path: the exact direct solve of
//     M U D + A U C = F            (stk/sylvester.hpp:58-65 heat_kron_op)
// through the tensor generalized eigenbasis, i.e. solve_projected_heat_with
// (stk/sylvester.hpp:117-142) with X = X_x (x) X_y (x) X_z:
//   K2  forward transforms  G~ = X^T F      (:126)    -> batched DMMA GEMMs per axis
//                                                        (dense backend), or FP64 fast
//                                                        sine transforms (P1_DST backend:
//                                                        dst.cuh, dst_half.cuh)
//   K3  per-mode recurrence (D + lambda_i C)^T y_i = g~_i   (:128-140) -> mode-parallel scan
//                                                        (heat_scan.cuh)
//   K2  inverse transforms  U = X Y~        (:141)
// and the K1 operator/residual kernel  out = M U D + A U C  (KronOp::apply, :32-38;
// heat_apply.cuh), the padded internal layout of the P1_DST device solve, the factored-load
// solve, and the host-buffer pipeline (stkg_heat_solve_host).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#include "common.cuh"
#include "dst.cuh"
#include "dst_half.cuh"
#include "heat_fused.cuh"  // K2b + K3: time-marching fused axis-0 pass
#include "heat_tridiag.cuh"  // K2e: time-marching line-solve axis-0 pass (uniform time grids)
#include "gemm_f64.cuh"
#include "heat_plan.cuh"
#include "heat_scan.cuh"   // K3: modal recurrences
#include "heat_apply.cuh"  // K1: operator / residual

using namespace stkg;

namespace {

// Sum interleaved partial pairs in a fixed order (deterministic).
__global__ void __launch_bounds__(256) sum_pairs_kernel(const double* partials, int64_t count,
                                                        double* result) {
  __shared__ double red[8];
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += 256) {
    a += partials[2 * i];
    b += partials[2 * i + 1];
  }
  a = block_sum<256>(a, red);
  b = block_sum<256>(b, red);
  if (threadIdx.x == 0) {
    result[0] = a;
    result[1] = b;
  }
}

__global__ void fill_uniform_kernel(double* dst, int64_t count, uint64_t seed, uint64_t stream,
                                    int64_t offset) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = uniform_pm1(seed, stream, uint64_t(offset + i));
}

}  // namespace

namespace stkg {
ModeLambda mode_lambda(const stkg_heat& h) {
  return ModeLambda{h.lam[0].p, h.ndim > 1 ? h.lam[1].p : nullptr,
                    h.ndim > 2 ? h.lam[2].p : nullptr, h.n[1], h.n[2], h.ndim};
}

}  // namespace stkg

namespace {
ModeWeight mode_weight(const stkg_heat& h) {
  if (h.transform != STKG_TRANSFORM_P1_DST) return ModeWeight{nullptr, nullptr, nullptr, 1, 1, 1};
  return ModeWeight{h.inv_mu[0].p, h.ndim > 1 ? h.inv_mu[1].p : nullptr,
                    h.ndim > 2 ? h.inv_mu[2].p : nullptr, h.n[1], h.n[2], h.ndim};
}

// The same over the padded internal layout (h.pitch > 0): n_last -> pitch, pad lanes get
// lambda 0 and weight 0 (their transformed data are zero, and stay zero).
int64_t padded_nx(const stkg_heat& h) { return h.nx / h.n[h.ndim - 1] * h.pitch; }
// The stream the DST / fused launchers use: the plan stream unless an overlapped schedule
// (run_chunk_padded_overlap) has redirected them.
cudaStream_t launch_stream(const stkg_heat& h) { return h.run_stream ? h.run_stream : h.stream; }
ModeLambda mode_lambda_padded(const stkg_heat& h) {
  if (h.ndim == 2) return ModeLambda{h.lam[0].p, h.lam_pad.p, nullptr, h.pitch, 1, 2};
  return ModeLambda{h.lam[0].p, h.lam[1].p, h.lam_pad.p, h.n[1], h.pitch, 3};
}
ModeWeight mode_weight_padded(const stkg_heat& h) {
  if (h.ndim == 2) return ModeWeight{h.inv_mu[0].p, h.inv_mu_pad.p, nullptr, h.pitch, 1, 2};
  return ModeWeight{h.inv_mu[0].p, h.inv_mu[1].p, h.inv_mu_pad.p, h.n[1], h.pitch, 3};
}

template <int L>
void launch_dst_strided(const stkg_heat& h, int a, const double* src, double* dst,
                        int64_t inner, int64_t outer) {
  using C = DstStridedLaunch<L>;
  static const bool configured = [] {
    STKG_CUDA_CHECK(cudaFuncSetAttribute(dst_strided_kernel<L>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::kSmem)));
    return true;
  }();
  (void)configured;
  int per_sm = 0;
  STKG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dst_strided_kernel<L>,
                                                                C::kThreads, C::kSmem));
  const int64_t nvec = outer * inner;
  const int64_t tiles = ceil_div(nvec, C::kG);
  const int64_t blocks = std::min<int64_t>(tiles, int64_t(num_sms()) * std::max(per_sm, 1));
  const double scale = std::sqrt(2.0 / static_cast<double>(h.n[a] + 1));
  dst_strided_kernel<L><<<static_cast<unsigned>(blocks), C::kThreads, C::kSmem, h.stream>>>(
      src, dst, h.n[a], inner, nvec, reinterpret_cast<const double2*>(h.twiddle[a].p), scale);
  STKG_CUDA_CHECK(cudaGetLastError());
}

template <int L>
void launch_dst(const stkg_heat& h, int a, const double* src, double* dst, int64_t inner,
                int64_t outer) {
  if (inner > 1) return launch_dst_strided<L>(h, a, src, dst, inner, outer);
  using C = DstLaunch<L>;
  static const bool configured = [] {
    STKG_CUDA_CHECK(cudaFuncSetAttribute(dst_axis_kernel<L>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::kSmem)));
    return true;
  }();
  (void)configured;
  int per_sm = 0;
  STKG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dst_axis_kernel<L>,
                                                                C::kThreads, C::kSmem));
  const int64_t nvec = outer * inner;
  const int64_t items = ceil_div(nvec, 2);
  const int64_t blocks = std::min<int64_t>(items, int64_t(num_sms()) * std::max(per_sm, 1));
  const double scale = std::sqrt(2.0 / static_cast<double>(h.n[a] + 1));
  dst_axis_kernel<L><<<static_cast<unsigned>(blocks), C::kThreads, C::kSmem, h.stream>>>(
      src, dst, h.n[a], inner, nvec, reinterpret_cast<const double2*>(h.twiddle[a].p), scale);
  STKG_CUDA_CHECK(cudaGetLastError());
}

// TMA descriptors: cuTensorMapEncodeTiled is a driver entry point, fetched through the
// runtime (the library links only cudart_static).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    STKG_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    STKG_REQUIRE(p && q == cudaDriverEntryPointSuccess, STKG_CUDA,
                 "cuTensorMapEncodeTiled entry point not available");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

CUtensorMapL2promotion tma_promotion() {  // STKG_TMA_PROMO = 0 / 64 / 128 / 256 (default 0)
  static const CUtensorMapL2promotion v = [] {
    const char* e = std::getenv("STKG_TMA_PROMO");
    const int b = e ? std::atoi(e) : 0;
    return b == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                    : b == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                               : b == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                         : CU_TENSOR_MAP_L2_PROMOTION_NONE;
  }();
  return v;
}

// Opt-in (STKG_TMA=1): measured 5% slower than the cp.async staging on the cfg3 strided
// passes (355 vs 336 us per 64 slices, same DRAM bytes, any box height or L2 promotion;
// tools/tma_promo.sh) -- a single thread's TMA boxes of 64-byte rows land later than 256
// threads' 16-byte cp.async copies of the same tile.
bool use_tma_strided() {
  static const bool on = [] {
    const char* e = std::getenv("STKG_TMA");
    return e && e[0] == '1';
  }();
  return on;
}

// Strided pass over [outer * n rows] x [inner columns] (row stride inner * 8 bytes) with
// the TMA kernel; tiles of 4 vector pairs = 8 columns of 64-byte rows.
template <int N>
void launch_dst_half_strided_tma(const stkg_heat& h, const double* src, double* dst,
                                 int64_t inner, int64_t outer, const double2* tw2,
                                 double scale) {
  using C = HalfStrided2Cfg<N, 4, false>;
  using TC = HalfStridedTmaCfg<N>;
  const int64_t nvec = outer * inner;
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer * (N - 1))};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(inner * sizeof(double))};
  const cuuint32_t box[2] = {8, TC::kBoxRows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = tensor_map_encoder()(
      &map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(src), dims, strides, box,
      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
      tma_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  STKG_REQUIRE(r == CUDA_SUCCESS, STKG_CUDA, "cuTensorMapEncodeTiled failed");
  static const int per_sm = [] {
    STKG_CUDA_CHECK(cudaFuncSetAttribute(dst_half_strided_tma_kernel<N>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(TC::kSmem)));
    int b = 0;
    STKG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &b, dst_half_strided_tma_kernel<N>, C::kThreads, TC::kSmem));
    return std::max(b, 1);
  }();
  const int64_t blocks = std::min<int64_t>(nvec / C::G, int64_t(num_sms()) * per_sm);
  dst_half_strided_tma_kernel<N><<<static_cast<unsigned>(blocks), C::kThreads, TC::kSmem,
                                   launch_stream(h)>>>(map, dst, inner, nvec, tw2, scale);
}

template <int N, int P, bool PF>
void launch_dst_half_strided2(const stkg_heat& h, const double* src, double* dst, int64_t inner,
                              int64_t nvec, const double2* tw2, double scale) {
  using C = HalfStrided2Cfg<N, P, PF>;
  static const int per_sm = [] {
    STKG_CUDA_CHECK(cudaFuncSetAttribute(dst_half_strided2_kernel<N, P, PF>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::kSmem)));
    int b = 0;
    STKG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &b, dst_half_strided2_kernel<N, P, PF>, C::kThreads, C::kSmem));
    return std::max(b, 1);
  }();
  const int64_t blocks = std::min<int64_t>(nvec / C::G, int64_t(num_sms()) * per_sm);
  dst_half_strided2_kernel<N, P, PF><<<static_cast<unsigned>(blocks), C::kThreads, C::kSmem,
                                       launch_stream(h)>>>(src, dst, inner, nvec, tw2, scale);
}

// Half-length kernels (dst_half.cuh) for N = n + 1 in [16, 1024].  Contiguous axis
// (inner == 1): vector g at src + g ld_src -> dst + g ld_dst (ld 0 = n).  Strided axes:
// dst_half_strided_kernel, or the 16-byte dst_half_strided2_kernel when `wide` (the padded
// layout: inner a multiple of its tile width, 16-byte aligned buffers).
// The contiguous pass of one-pair-per-CTA plans (N = 1024) takes its input by one bulk copy
// per pair (dst_half_bulk_kernel) instead of per-thread loads: bit-identical, cfg3 solve
// 10.60 -> 10.37 ms (same box, alternating runs).  STKG_DST_BULK=0 keeps the per-thread loads.
bool dst_bulk_input() {
  static const bool on = [] {
    const char* e = std::getenv("STKG_DST_BULK");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

template <int N>
void launch_dst_half(const stkg_heat& h, int a, const double* src, double* dst, int64_t inner,
                     int64_t outer, int64_t ld_src = 0, int64_t ld_dst = 0, bool wide = false) {
  const int64_t nvec = outer * inner;
  const double scale = std::sqrt(2.0 / static_cast<double>(N));
  const double2* tw2 = reinterpret_cast<const double2*>(h.twiddle[a].p);
  if (inner == 1) {
    using C = HalfCfg<N>;
    static const int per_sm = [] {
      STKG_CUDA_CHECK(cudaFuncSetAttribute(dst_half_kernel<N>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(C::kSmem)));
      int b = 0;
      STKG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, dst_half_kernel<N>,
                                                                    C::kThreads, C::kSmem));
      return std::max(b, 1);
    }();
    const int64_t blocks = std::min<int64_t>(ceil_div(nvec, 2 * C::F), int64_t(num_sms()) * per_sm);
    const int64_t lds = ld_src > 0 ? ld_src : N - 1, ldd = ld_dst > 0 ? ld_dst : N - 1;
    if (h.run_ticket) {
      static const bool dyn_configured = [] {
        STKG_CUDA_CHECK(cudaFuncSetAttribute(dst_half_kernel<N, true>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(C::kSmem)));
        return true;
      }();
      (void)dyn_configured;
      dst_half_kernel<N, true><<<static_cast<unsigned>(blocks), C::kThreads, C::kSmem,
                                 launch_stream(h)>>>(src, dst, nvec, tw2, scale, lds, ldd,
                                                     h.run_ticket);
    } else if (C::F == 1 && dst_bulk_input() && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
               src != dst) {
      if constexpr (C::F == 1) {
        constexpr size_t bsmem = C::kSmem + (STKG_DST_BULK_SEP ? size_t(16) * N : 0);
        static const int bulk_per_sm = [] {
          STKG_CUDA_CHECK(cudaFuncSetAttribute(dst_half_bulk_kernel<N>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(bsmem)));
          int b = 0;
          STKG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
              &b, dst_half_bulk_kernel<N>, C::kThreads, bsmem));
          return std::max(b, 1);
        }();
        const int64_t bblocks =
            std::min<int64_t>(ceil_div(nvec, 2), int64_t(num_sms()) * bulk_per_sm);
        dst_half_bulk_kernel<N><<<static_cast<unsigned>(bblocks), C::kThreads, bsmem,
                                  launch_stream(h)>>>(src, dst, nvec, tw2, scale, lds, ldd);
      }
    } else {
      dst_half_kernel<N><<<static_cast<unsigned>(blocks), C::kThreads, C::kSmem,
                           launch_stream(h)>>>(src, dst, nvec, tw2, scale, lds, ldd);
    }
  } else if (wide && inner % HalfStrided2Cfg<N>::G == 0) {
    if constexpr (N / half_v<N>() >= 32) {  // tiles of 4 pairs: optional TMA staging
      if (use_tma_strided() && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
          outer * (N - 1) < (int64_t(1) << 31) && inner < (int64_t(1) << 31)) {
        launch_dst_half_strided_tma<N>(h, src, dst, inner, outer, tw2, scale);
        STKG_CUDA_CHECK(cudaGetLastError());
        return;
      }
    }
    if constexpr (N == 1024) {  // tuning variants: STKG_HALF2 = pairs * 10 + prefetch
      static const int var = [] {
        const char* e = std::getenv("STKG_HALF2");
        return e ? std::atoi(e) : 40;
      }();
      switch (var) {
        case 41: return launch_dst_half_strided2<N, 4, true>(h, src, dst, inner, nvec, tw2, scale);
        case 20: return launch_dst_half_strided2<N, 2, false>(h, src, dst, inner, nvec, tw2, scale);
        case 21: return launch_dst_half_strided2<N, 2, true>(h, src, dst, inner, nvec, tw2, scale);
        default: break;
      }
    }
    launch_dst_half_strided2<N, half2_pairs<N>(), false>(h, src, dst, inner, nvec, tw2, scale);
  } else {
    using C = HalfStridedCfg<N>;
    static const int per_sm = [] {
      STKG_CUDA_CHECK(cudaFuncSetAttribute(dst_half_strided_kernel<N>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(C::kSmem)));
      int b = 0;
      STKG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &b, dst_half_strided_kernel<N>, C::kThreads, C::kSmem));
      return std::max(b, 1);
    }();
    const int64_t blocks = std::min<int64_t>(ceil_div(nvec, C::G), int64_t(num_sms()) * per_sm);
    dst_half_strided_kernel<N><<<static_cast<unsigned>(blocks), C::kThreads, C::kSmem, launch_stream(h)>>>(
        src, dst, inner, nvec, tw2, scale);
  }
  STKG_CUDA_CHECK(cudaGetLastError());
}

bool padded_layout_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("STKG_PAD");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool use_dst_half() {
  static const bool on = [] {
    const char* e = std::getenv("STKG_DST_HALF");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Half-length DST pass with explicit leading dimensions (contiguous axis) or the 16-byte
// strided kernel (wide); false when N = n_a + 1 has no half-length kernel.
bool dst_half_pass(const stkg_heat& h, int a, const double* src, double* dst, int64_t inner,
                   int64_t outer, int64_t ld_src = 0, int64_t ld_dst = 0, bool wide = false) {
  switch (h.n[a] + 1) {
    // N = 2048 keeps the padded 2N kernel: the half-length recurrence's sqrt(N) error
    // growth costs 1D n = 2047 the 1e-10 residual gate (3e-10 measured)
    case 16: launch_dst_half<16>(h, a, src, dst, inner, outer, ld_src, ld_dst, wide); return true;
    case 32: launch_dst_half<32>(h, a, src, dst, inner, outer, ld_src, ld_dst, wide); return true;
    case 64: launch_dst_half<64>(h, a, src, dst, inner, outer, ld_src, ld_dst, wide); return true;
    case 128: launch_dst_half<128>(h, a, src, dst, inner, outer, ld_src, ld_dst, wide); return true;
    case 256: launch_dst_half<256>(h, a, src, dst, inner, outer, ld_src, ld_dst, wide); return true;
    case 512: launch_dst_half<512>(h, a, src, dst, inner, outer, ld_src, ld_dst, wide); return true;
    case 1024: launch_dst_half<1024>(h, a, src, dst, inner, outer, ld_src, ld_dst, wide); return true;
    default: return false;
  }
}

// Time-marching fused pass over axis 0 of the padded layout (heat_fused.cuh): forward
// transform, recurrence and inverse transform of every slice of S in one kernel.
template <int N, int P = fused_pairs<N>(), bool CS = false, bool TMA = false,
          int V = half2_v<N>(), int MB = 1, int MAXR = 0>
void launch_fused_axis0(const stkg_heat& h, double* S, int64_t inner, int64_t ntc, int64_t l0) {
  using C = FusedCfg<N, P, CS, TMA, V, MB>;
  static_assert(MAXR == 0, "register-capped instantiation removed (DESIGN.md K2c)");
  auto kern = heat_fused_axis0_kernel<N, P, CS, TMA, V, MB>;
  static const bool configured = [kern] {
    STKG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::kSmem)));
    return true;
  }();
  (void)configured;
  CUtensorMap map;
  std::memset(&map, 0, sizeof map);
  if constexpr (TMA) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner),
                                static_cast<cuuint64_t>(ntc * h.n[0])};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(inner * sizeof(double))};
    const cuuint32_t box[2] = {8, C::kBoxRows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = tensor_map_encoder()(
        &map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, S, dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, tma_promotion(),
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    STKG_REQUIRE(r == CUDA_SUCCESS, STKG_CUDA, "cuTensorMapEncodeTiled failed");
  }
  const int64_t tiles = inner / C::G;
  const double scale = std::sqrt(2.0 / static_cast<double>(N));
  kern<<<static_cast<unsigned>(tiles), C::kThreads, C::kSmem,
                                              launch_stream(h)>>>(
      map, S, inner, h.n[0] * inner, ntc, l0, reinterpret_cast<const double2*>(h.twiddle[0].p),
      scale, h.lam[0].p, h.inv_mu[0].p, h.lam_col.p, h.w_col.p, h.d_diag.p, h.d_sup.p,
      h.c_diag.p, h.c_sup.p, h.carry.p);
  STKG_CUDA_CHECK(cudaGetLastError());
}

// Time-marching line-solve pass over axis 0 (heat_tridiag.cuh): one tridiagonal solve per
// column and slice instead of the two transforms; plans with h.tri_ok.
template <int N, int P, int ST = 3>
void launch_tridiag_axis0(const stkg_heat& h, double* S, int64_t inner, int64_t ntc, int64_t l0) {
  using C = TriCfg<N, P, ST>;
  auto kern = heat_tridiag_axis0_kernel<N, P, ST>;
  static const bool configured = [kern] {
    STKG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::kSmem)));
    return true;
  }();
  (void)configured;
  const int64_t tiles = inner / C::G;
  const double ds = h.nt > 1 ? h.d_sup_h[0] : 0.0, cs = h.nt > 1 ? h.c_sup_h[0] : 0.0;
  kern<<<static_cast<unsigned>(tiles), C::kThreads, C::kSmem, launch_stream(h)>>>(
      S, inner, h.n[0] * inner, ntc, l0, h.tri_iw.p, h.lam_col.p, h.w_col.p, h.d_diag_h[0], ds,
      h.c_diag_h[0], cs, h.tri_md, h.tri_mo, h.tri_ad, h.tri_ao, h.carry.p);
  STKG_CUDA_CHECK(cudaGetLastError());
}

// STKG_TRI_V: 1 (default) = TMA tile staging and stores, 0 = cp.async staging.
int tri_variant() {
  static const int v = [] {
    const char* e = std::getenv("STKG_TRI_V");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

template <int N, int P, bool UNI, bool GUARD>
void launch_tridiag_tma_u(const stkg_heat& h, double* S, int64_t inner, int64_t ntc, int64_t l0) {
  using C = TriTmaCfg<N, P>;
  auto kern = heat_tridiag_tma_kernel<N, P, UNI, GUARD>;
  static const bool configured = [kern] {
    STKG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::kSmem)));
    return true;
  }();
  (void)configured;
  // the launch's slices as [ntc][n_0][inner]: rows >= n_0 are out of bounds (zero-filled on
  // load, clipped on store)
  CUtensorMap map;
  std::memset(&map, 0, sizeof map);
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(h.n[0]),
                              static_cast<cuuint64_t>(ntc)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(inner * sizeof(double)),
                                 static_cast<cuuint64_t>(h.n[0] * inner * sizeof(double))};
  const cuuint32_t box[3] = {C::CW / 8, C::BR, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = tensor_map_encoder()(
      &map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, S, dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE,
      C::CW == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, tma_promotion(),
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  STKG_REQUIRE(r == CUDA_SUCCESS, STKG_CUDA, "cuTensorMapEncodeTiled failed (line-solve pass)");
  const int64_t tiles = inner / C::G;
  const double ds = h.nt > 1 ? h.d_sup_h[0] : 0.0, cs = h.nt > 1 ? h.c_sup_h[0] : 0.0;
  kern<<<static_cast<unsigned>(tiles), C::kThreads, C::kSmem, launch_stream(h)>>>(
      map, inner, ntc, l0, h.lam_col.p, h.w_col.p, h.d_diag_h[0], ds, h.c_diag_h[0], cs, h.tri_md,
      h.tri_mo, h.tri_ad, h.tri_ao, h.carry.p, h.d_diag.p, h.d_sup.p, h.c_diag.p, h.c_sup.p);
  STKG_CUDA_CHECK(cudaGetLastError());
}

template <int N, int P>
void launch_tridiag_tma(const stkg_heat& h, double* S, int64_t inner, int64_t ntc, int64_t l0) {
  // STKG_TRI_GUARD: 0 / 1 forces the unguarded / guarded kernel; unset: guarded when the
  // tiles fill most of the GPU (the HBM-bound regime, see heat_tridiag_tma_kernel)
  static const int force = [] {
    const char* e = std::getenv("STKG_TRI_GUARD");
    return e ? std::atoi(e) : -1;
  }();
  const bool guard = force >= 0 ? force != 0 : inner / TriTmaCfg<N, P>::G >= (3 * num_sms()) / 4;
  if (!h.uniform_time) return launch_tridiag_tma_u<N, P, false, false>(h, S, inner, ntc, l0);
  if (guard) return launch_tridiag_tma_u<N, P, true, true>(h, S, inner, ntc, l0);
  return launch_tridiag_tma_u<N, P, true, false>(h, S, inner, ntc, l0);
}

// Columns per line-solve tile for axis-0 length n0 (0: no such kernel for that length).
int64_t tri_tile_cols(int64_t n0) {
  switch (n0 + 1) {
    case 64: return 64;
    case 128: return 64;
    case 256: return 32;
    case 512: return 16;
    case 1024: return 8;
    default: return 0;
  }
}

void tridiag_axis0(const stkg_heat& h, double* S, int64_t inner, int64_t ntc, int64_t l0) {
  const bool tma_ok = (reinterpret_cast<uintptr_t>(S) & 15) == 0 && inner < (int64_t(1) << 31) &&
                      ntc < (int64_t(1) << 31);
  STKG_REQUIRE(tri_variant() == 0 || tma_ok, STKG_ARGUMENT,
               "line-solve pass: scratch not addressable by a tensor map");
  if (tri_variant() != 0) {
    switch (h.n[0] + 1) {
      case 64: return launch_tridiag_tma<64, 32>(h, S, inner, ntc, l0);
      case 128: return launch_tridiag_tma<128, 32>(h, S, inner, ntc, l0);
      case 256: return launch_tridiag_tma<256, 16>(h, S, inner, ntc, l0);
      case 512: return launch_tridiag_tma<512, 8>(h, S, inner, ntc, l0);
      case 1024: return launch_tridiag_tma<1024, 4>(h, S, inner, ntc, l0);
      default: break;
    }
  }
  switch (h.n[0] + 1) {
    case 64: return launch_tridiag_axis0<64, 32>(h, S, inner, ntc, l0);
    case 128: return launch_tridiag_axis0<128, 32>(h, S, inner, ntc, l0);
    case 256: return launch_tridiag_axis0<256, 16>(h, S, inner, ntc, l0);
    case 512: return launch_tridiag_axis0<512, 8>(h, S, inner, ntc, l0);
    case 1024: return launch_tridiag_axis0<1024, 4>(h, S, inner, ntc, l0);
    default: throw Error(STKG_ARGUMENT, "line-solve pass: unsupported axis length");
  }
}

bool use_tridiag(const stkg_heat& h, int64_t inner) {
  const int64_t G = tri_tile_cols(h.n[0]);
  return h.tri_ok && G > 0 && inner % G == 0;
}

// Columns per fused tile for axis-0 length n0 (0: no fused kernel for that length).
int64_t fused_tile_cols(int64_t n0) {
  switch (n0 + 1) {
    case 16: return FusedCfg<16, fused_pairs<16>()>::G;
    case 32: return FusedCfg<32, fused_pairs<32>()>::G;
    case 64: return FusedCfg<64, fused_pairs<64>()>::G;
    case 128: return FusedCfg<128, fused_pairs<128>()>::G;
    case 256: return FusedCfg<256, fused_pairs<256>()>::G;
    case 512: return FusedCfg<512, fused_pairs<512>()>::G;
    case 1024: {
      const char* e = std::getenv("STKG_FUSED_P");
      return e ? 2 * std::atoi(e) : FusedCfg<1024, fused_pairs<1024>()>::G;
    }
    default: return 0;
  }
}

// STKG_FUSED=0: the separate strided passes + scan kernel; 1: the fused pass whenever the
// tile geometry allows; unset: the fused pass when it has at least half a CTA per SM.
int fused_mode() {
  static const int m = [] {
    const char* e = std::getenv("STKG_FUSED");
    return e ? std::atoi(e) : -1;
  }();
  return m;
}

// Columns per tile of whichever time-marching axis-0 pass the plan runs.
int64_t axis0_tile_cols(const stkg_heat& h, int64_t inner) {
  return use_tridiag(h, inner) ? tri_tile_cols(h.n[0]) : fused_tile_cols(h.n[0]);
}

bool use_fused_axis0(const stkg_heat& h, int64_t inner) {
  if (h.pitch <= 0 || h.lam_col.p == nullptr) return false;
  const int64_t G = axis0_tile_cols(h, inner);
  if (G == 0 || inner % G != 0) return false;
  const int m = fused_mode();
  if (m == 0) return false;
  if (m > 0) return true;
  // the line-solve pass costs ~2 us per slice whatever the tile count, so it pays from 32 tiles
  // on (measured: 2D 511^2 x 1024 4.52 vs 5.56 ms, 3D 63^3 x 512 3.34 vs 3.91 ms; 8 tiles at
  // 255^2 lose 2.7 vs 1.5 ms); the fused transform pass needs half a CTA per SM
  if (use_tridiag(h, inner)) return inner / G >= 32;
  return inner / G >= num_sms() / 2;
}

void fused_axis0(const stkg_heat& h, double* S, int64_t inner, int64_t ntc, int64_t l0) {
  if (use_tridiag(h, inner)) return tridiag_axis0(h, S, inner, ntc, l0);
  switch (h.n[0] + 1) {
    case 16: return launch_fused_axis0<16>(h, S, inner, ntc, l0);
    case 32: return launch_fused_axis0<32>(h, S, inner, ntc, l0);
    case 64: return launch_fused_axis0<64>(h, S, inner, ntc, l0);
    case 128: return launch_fused_axis0<128>(h, S, inner, ntc, l0);
    case 256: return launch_fused_axis0<256>(h, S, inner, ntc, l0);
    case 512: return launch_fused_axis0<512>(h, S, inner, ntc, l0);
    case 1024: {
      // tuning knob STKG_FUSED_P: vector pairs per tile (1, 2 or 4)
      static const int pp = [] {
        const char* e = std::getenv("STKG_FUSED_P");
        return e ? std::atoi(e) : fused_pairs<1024>();
      }();
      // STKG_FUSED_V: 1 = carries in shared memory, 2 = TMA tile staging (tiles of 4 pairs),
      // 8 = 8 values per thread (128-thread FFTs)
      static const int fv = [] {
        const char* e = std::getenv("STKG_FUSED_V");
        return e ? std::atoi(e) : 0;
      }();
      if (pp == 1) return launch_fused_axis0<1024, 1>(h, S, inner, ntc, l0);
      if (pp == 2) return launch_fused_axis0<1024, 2>(h, S, inner, ntc, l0);
      const bool tma_ok = (reinterpret_cast<uintptr_t>(S) & 15) == 0 &&
                          ntc * h.n[0] < (int64_t(1) << 31) && inner < (int64_t(1) << 31);
      if (fv == 8) return launch_fused_axis0<1024, 4, false, false, 8>(h, S, inner, ntc, l0);
      switch (tma_ok ? fv : fv & 1) {
        case 1: return launch_fused_axis0<1024, 4, true, false>(h, S, inner, ntc, l0);
        case 2: return launch_fused_axis0<1024, 4, false, true>(h, S, inner, ntc, l0);
        case 3: return launch_fused_axis0<1024, 4, true, true>(h, S, inner, ntc, l0);
        default: return launch_fused_axis0<1024>(h, S, inner, ntc, l0);
      }
    }
    default: throw Error(STKG_ARGUMENT, "fused pass: unsupported axis length");
  }
}

void dst_pass(const stkg_heat& h, int a, const double* src, double* dst, int64_t inner,
              int64_t outer) {
  // The half-length kernels trade accuracy for speed (their odd outputs are a prefix sum):
  // measured relres 2.6e-12 (2D, n = 1023) and 7e-13 (2D 511) but 5e-11 for 1D n = 1023,
  // too close to the 1e-10 gate -- so 1D plans keep the padded kernels.
  if (use_dst_half() && h.ndim >= 2 && dst_half_pass(h, a, src, dst, inner, outer)) return;
  switch (2 * (h.n[a] + 1)) {
    case 32: return launch_dst<32>(h, a, src, dst, inner, outer);
    case 64: return launch_dst<64>(h, a, src, dst, inner, outer);
    case 128: return launch_dst<128>(h, a, src, dst, inner, outer);
    case 256: return launch_dst<256>(h, a, src, dst, inner, outer);
    case 512: return launch_dst<512>(h, a, src, dst, inner, outer);
    case 1024: return launch_dst<1024>(h, a, src, dst, inner, outer);
    case 2048: return launch_dst<2048>(h, a, src, dst, inner, outer);
    case 4096: return launch_dst<4096>(h, a, src, dst, inner, outer);
    default: throw Error(STKG_ARGUMENT, "P1_DST transform: n + 1 must be a power of two in [16, 2048]");
  }
}

// One axis transform over a block of ntc time slices.  Axis a with inner extent
// I = prod_{b>a} n_b: the fastest axis (I == 1) is a left product  Op * data(n_a x rest);
// every other axis is a batched right product  data_b(I x n_a) * Op'  (SURVEY Appendix A:
// G~_l = X_y^T F_l X_x in column-major slices).
struct ProfScope {  // records a begin/end event pair around one launch when profiling
  stkg_heat& h;
  int cls;
  cudaEvent_t e1 = nullptr;
  ProfScope(stkg_heat& hh, int c) : h(hh), cls(c) {
    if (!h.prof_on) return;
    cudaEvent_t e0;
    STKG_CUDA_CHECK(cudaEventCreate(&e0));
    STKG_CUDA_CHECK(cudaEventCreate(&e1));
    STKG_CUDA_CHECK(cudaEventRecord(e0, h.stream));
    h.prof_ev[cls].push_back(e0);
    h.prof_ev[cls].push_back(e1);
  }
  ~ProfScope() {
    if (!h.prof_on) return;
    cudaEventRecord(e1, h.stream);
    h.prof_launches[cls]++;
  }
};

}  // namespace

namespace stkg {
void axis_pass(stkg_heat& h, int a, bool forward, const double* src, double* dst,
               int64_t ntc) {
  int64_t inner = 1, outer = ntc;
  for (int b = a + 1; b < h.ndim; ++b) inner *= h.n[b];
  for (int b = 0; b < a; ++b) outer *= h.n[b];
  const int64_t na = h.n[a];
  if (h.transform == STKG_TRANSFORM_P1_DST) {  // X = S diag(mu^-1/2): S is its own inverse
    ProfScope ps(h, 0);
    dst_pass(h, a, src, dst, inner, outer);
    return;
  }
  GemmProblem p;
  if (inner == 1) {
    p.M = na;
    p.K = na;
    p.N = outer;
    p.A = forward ? h.XT[a].p : h.X[a].p;
    p.lda = na;
    p.B = src;
    p.ldb = na;
    p.C = dst;
    p.ldc = na;
  } else {
    p.M = inner;
    p.K = na;
    p.N = na;
    p.batch = outer;
    p.A = src;
    p.lda = inner;
    p.strideA = inner * na;
    p.B = forward ? h.X[a].p : h.XT[a].p;
    p.ldb = na;
    p.C = dst;
    p.ldc = inner;
    p.strideC = inner * na;
  }
  ProfScope ps(h, 0);
  launch_gemm(p, EpiStore{}, h.stream);
}

}  // namespace stkg

namespace {
// STKG_OVERLAP: time chunks of the overlapped 2D schedule (0 or 1: off).
int overlap_chunks() {
  static const int k = [] {
    const char* e = std::getenv("STKG_OVERLAP");
    return e ? std::atoi(e) : 4;
  }();
  return k;
}

// 2D plans whose fused axis-0 pass has fewer tiles than the GPU has SMs (cfg3: 128 tiles on
// 148 SMs) leave SMs idle for the whole fused pass.  This schedule cuts time into K chunks and
// runs, on a low-priority stream, the contiguous forward pass of later chunks and the
// contiguous inverse pass of earlier ones while the fused pass of chunk c runs on a
// high-priority stream:
//   lo:  C1(0) C1(1) C1(2) [X0] C2(0) C1(3) [X1] C2(1) [X2] C2(2) [X3] C2(3)
//   hi:  [C1(0)] X(0) [C1(1)] X(1) [C1(2)] X(2) [C1(3)] X(3)
// (brackets: event waits).  The fused pass holds all registers of its SMs, so the contiguous
// CTAs land only on the idle SMs while it runs; they take their items from a ticket counter
// (dst_half_kernel's dynamic mode), so the items of CTAs that are not yet resident are not
// stranded behind the fused pass.  The recurrence carries cross chunks through h.carry
// (X(c) follows X(c-1) on the same stream).  Same arithmetic as run_chunk_padded.
void run_chunk_padded_overlap(stkg_heat& h, const double* F, double* U, double* S, int64_t l0,
                              int64_t ntc, int K, int64_t inner0) {
  const int64_t nl = h.n[1], P = h.pitch, lines = h.nx / nl, sp = padded_nx(h);
  if (!h.s_hi) {
    int least = 0, greatest = 0;
    STKG_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    STKG_CUDA_CHECK(cudaStreamCreateWithPriority(&h.s_hi, cudaStreamNonBlocking, greatest));
    STKG_CUDA_CHECK(cudaStreamCreateWithPriority(&h.s_lo, cudaStreamNonBlocking, least));
  }
  const size_t nev = 2 * size_t(K) + 3;
  while (h.ov_ev.size() < nev) {
    cudaEvent_t e;
    STKG_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    h.ov_ev.push_back(e);
  }
  if (h.tickets_n < 2 * K) {
    if (h.tickets) STKG_CUDA_CHECK(cudaFree(h.tickets));
    STKG_CUDA_CHECK(cudaMalloc(&h.tickets, 2 * K * sizeof(unsigned long long)));
    h.tickets_n = 2 * K;
  }
  cudaEvent_t* ev_c1 = h.ov_ev.data();
  cudaEvent_t* ev_x = ev_c1 + K;
  cudaEvent_t ev_start = ev_x[K], ev_lo = ev_x[K + 1], ev_hi = ev_x[K + 2];
  STKG_CUDA_CHECK(cudaEventRecord(ev_start, h.stream));
  STKG_CUDA_CHECK(cudaStreamWaitEvent(h.s_hi, ev_start, 0));
  STKG_CUDA_CHECK(cudaStreamWaitEvent(h.s_lo, ev_start, 0));
  STKG_CUDA_CHECK(cudaMemsetAsync(h.tickets, 0, 2 * K * sizeof(unsigned long long), h.s_lo));
  // even slice counts per chunk: every chunk then starts at an even vector index, so the
  // contiguous passes pair the same vectors in one complex FFT as the unchunked pass does
  // (bit-identical results; tests/test_heat_gpu.py::test_overlapped_schedule_bit_identical)
  const int64_t chunk = ((ntc + K - 1) / K + 1) / 2 * 2;
  auto c0 = [&](int c) { return std::min<int64_t>(ntc, c * chunk); };
  while (K > 1 && c0(K - 1) >= ntc) --K;  // rounding up may leave trailing chunks empty
  auto len = [&](int c) { return c0(c + 1) - c0(c); };
  auto C1 = [&](int c) {
    h.run_stream = h.s_lo;
    h.run_ticket = h.tickets + c;
    dst_half_pass(h, 1, F + c0(c) * h.nx, S + c0(c) * sp, 1, lines * len(c), nl, P);
    STKG_CUDA_CHECK(cudaEventRecord(ev_c1[c], h.s_lo));
  };
  auto C2 = [&](int c) {
    STKG_CUDA_CHECK(cudaStreamWaitEvent(h.s_lo, ev_x[c], 0));
    h.run_stream = h.s_lo;
    h.run_ticket = h.tickets + K + c;
    dst_half_pass(h, 1, S + c0(c) * sp, U + c0(c) * h.nx, 1, lines * len(c), P, nl);
  };
  auto X = [&](int c) {
    STKG_CUDA_CHECK(cudaStreamWaitEvent(h.s_hi, ev_c1[c], 0));
    h.run_stream = h.s_hi;
    h.run_ticket = nullptr;
    fused_axis0(h, S + c0(c) * sp, inner0, len(c), l0 + c0(c));
    STKG_CUDA_CHECK(cudaEventRecord(ev_x[c], h.s_hi));
  };
  try {
    // host enqueue order keeps every event record ahead of its waits
    C1(0);
    X(0);
    if (K > 1) C1(1);
    for (int c = 1; c < K; ++c) {
      X(c);
      if (c + 1 < K) C1(c + 1);
      C2(c - 1);
    }
    C2(K - 1);
  } catch (...) {
    // rejoin whatever was enqueued before the error, so later work on the plan stream
    // cannot overtake it (best effort: the error being reported is the first one)
    h.run_stream = nullptr;
    h.run_ticket = nullptr;
    cudaEventRecord(ev_lo, h.s_lo);
    cudaEventRecord(ev_hi, h.s_hi);
    cudaStreamWaitEvent(h.stream, ev_lo, 0);
    cudaStreamWaitEvent(h.stream, ev_hi, 0);
    throw;
  }
  h.run_stream = nullptr;
  h.run_ticket = nullptr;
  STKG_CUDA_CHECK(cudaEventRecord(ev_lo, h.s_lo));
  STKG_CUDA_CHECK(cudaEventRecord(ev_hi, h.s_hi));
  STKG_CUDA_CHECK(cudaStreamWaitEvent(h.stream, ev_lo, 0));
  STKG_CUDA_CHECK(cudaStreamWaitEvent(h.stream, ev_hi, 0));
}

}  // namespace

namespace {
// Full solve of ntc time slices starting at l0 (carry holds y_{l0-1} when l0 > 0), P1_DST
// 2D/3D plans (h.pitch > 0).  Every intermediate lives in S in the padded layout (fastest
// axis at pitch N = n + 1, pad entries zero), so that the strided passes run the 16-byte
// kernel in place:  F -(fastest axis)-> S -(other axes, in place)-> S -(scan)-> S
// -(other axes)-> S -(fastest axis)-> U.
void run_chunk_padded(stkg_heat& h, const double* F, double* U, double* S, int64_t l0,
                      int64_t ntc) {
  const int d = h.ndim, last = d - 1;
  const int64_t nl = h.n[last], P = h.pitch;
  const int64_t lines = h.nx / nl * ntc;  // vectors along the fastest axis
  auto strided = [&](int a) {
    int64_t inner = P, outer = ntc;
    for (int b = a + 1; b < last; ++b) inner *= h.n[b];
    for (int b = 0; b < a; ++b) outer *= h.n[b];
    ProfScope ps(h, 0);
    dst_half_pass(h, a, S, S, inner, outer, 0, 0, true);
  };
  int64_t inner0 = P;  // columns of axis 0
  for (int b = 1; b < last; ++b) inner0 *= h.n[b];
  const bool fused = use_fused_axis0(h, inner0);
  // (the line-solve pass is an HBM stream: running the contiguous passes beside it only
  // splits the bandwidth -- measured 12.0 vs 10.8 ms on cfg3 -- so it keeps the plain order)
  static const bool overlap_line = [] {  // STKG_OVERLAP_LINE=1: the overlap for line-solve plans too
    const char* e = std::getenv("STKG_OVERLAP_LINE");
    return e && std::atoi(e) != 0;
  }();
  if (fused && (overlap_line || !use_tridiag(h, inner0)) && d == 2 && !h.prof_on &&
      overlap_chunks() > 1 &&
      ntc >= 8 * overlap_chunks() && inner0 / axis0_tile_cols(h, inner0) < num_sms()) {
    run_chunk_padded_overlap(h, F, U, S, l0, ntc, overlap_chunks(), inner0);
    return;
  }
  {
    ProfScope ps(h, 0);
    dst_half_pass(h, last, F, S, 1, lines, nl, P);
  }
  if (fused) {
    // axes last-1 .. 1 forward, then axis 0 forward + recurrence + inverse marching in time
    for (int a = last - 1; a >= 1; --a) strided(a);
    {
      ProfScope ps(h, 1);  // the fused pass runs the modal recurrence (class 1)
      fused_axis0(h, S, inner0, ntc, l0);
    }
    for (int a = 1; a < last; ++a) strided(a);
  } else {
    for (int a = last - 1; a >= 0; --a) strided(a);
    {
      const int64_t nxp = padded_nx(h);
      ProfScope ps(h, 1);
      launch_scan(h, S, nxp, ntc, l0, mode_lambda_padded(h), mode_weight_padded(h));
      STKG_CUDA_CHECK(cudaGetLastError());
    }
    for (int a = 0; a < last; ++a) strided(a);
  }
  {
    ProfScope ps(h, 0);
    dst_half_pass(h, last, S, U, 1, lines, P, nl);
  }
}

// The inverse passes of run_chunk_padded alone (factored solve): S (padded, modified in
// place) -> U.
void inverse_passes_padded(stkg_heat& h, double* S, double* U, int64_t ntc) {
  const int d = h.ndim, last = d - 1;
  const int64_t nl = h.n[last], P = h.pitch;
  for (int a = 0; a < last; ++a) {
    int64_t inner = P, outer = ntc;
    for (int b = a + 1; b < last; ++b) inner *= h.n[b];
    for (int b = 0; b < a; ++b) outer *= h.n[b];
    ProfScope ps(h, 0);
    dst_half_pass(h, a, S, S, inner, outer, 0, 0, true);
  }
  ProfScope ps(h, 0);
  dst_half_pass(h, last, S, U, 1, h.nx / nl * ntc, P, nl);
}

// Full solve of ntc time slices starting at l0 (carry holds y_{l0-1} when l0 > 0).
// Passes alternate between U and S so that the last inverse pass lands in U.
void run_chunk(stkg_heat& h, const double* F, double* U, double* S, int64_t l0, int64_t ntc) {
  if (h.pitch > 0) return run_chunk_padded(h, F, U, S, l0, ntc);
  const int d = h.ndim, passes = 2 * d;
  const double* src = F;
  int k = 0;
  auto next_dst = [&](int kk) { return ((passes - kk) % 2 == 0) ? U : S; };
  for (int a = d - 1; a >= 0; --a) {  // forward, fastest axis first
    double* dst = next_dst(++k);
    axis_pass(h, a, true, src, dst, ntc);
    src = dst;
  }
  {
    double* Y = const_cast<double*>(src);
    const int64_t blocks = ceil_div(h.nx, 256);
    ProfScope ps(h, 1);
    (void)blocks;
    launch_scan(h, Y, h.nx, ntc, l0, mode_lambda(h), mode_weight(h));
    STKG_CUDA_CHECK(cudaGetLastError());
  }
  for (int a = 0; a < d; ++a) {  // inverse, slowest axis first
    double* dst = next_dst(++k);
    axis_pass(h, a, false, src, dst, ntc);
    src = dst;
  }
}

// Slices per L2-resident sub-chunk.  Running all passes of a few time slices back to back
// keeps the intermediate slices (the U sub-chunk and the scratch) in the 126 MB L2, so HBM
// sees F once and U once (16 B/unknown) instead of 16 B/unknown per pass.  The recurrence
// carries its state across sub-chunks (heat_scan_kernel's carry).  STKG_L2_CHUNK_MB
// overrides the working-set budget (0 = one chunk over all of n_t).
int64_t l2_chunk_slices(const stkg_heat& h) {
  static const long budget_mb = [] {
    const char* e = std::getenv("STKG_L2_CHUNK_MB");
    return e ? std::atol(e) : -1L;
  }();
  long mb = budget_mb;
  if (mb < 0) mb = 0;  // measured: sub-chunking loses to whole-n_t passes (DESIGN K2b)
  if (mb == 0) return h.nt;
  const int64_t per_slice = 2 * h.nx * static_cast<int64_t>(sizeof(double));  // U + scratch
  return std::min<int64_t>(h.nt, std::max<int64_t>(1, (int64_t(mb) << 20) / per_slice));
}

// F, U: slices [l0, l0 + ntc) (already offset).  Uses h.scratch (grown to one sub-chunk).
void solve_range(stkg_heat& h, const double* F, double* U, int64_t l0, int64_t ntc) {
  const int64_t tc = std::min(l2_chunk_slices(h), ntc);
  const int64_t slice = h.pitch > 0 ? padded_nx(h) : h.nx;
  if (h.scratch.n < static_cast<size_t>(slice * tc)) {
    STKG_CUDA_CHECK(cudaStreamSynchronize(h.stream));
    h.scratch.alloc(slice * tc);
  }
  for (int64_t j = 0; j < ntc; j += tc) {
    const int64_t m = std::min(tc, ntc - j);
    run_chunk(h, F + j * h.nx, U + j * h.nx, h.scratch.p, l0 + j, m);
  }
}

// Inverse transforms only, from Y (which must be the buffer the first pass does not
// write) into U; used by the factored solve.
void inverse_passes(stkg_heat& h, const double* Y, double* U, double* S, int64_t ntc) {
  const int d = h.ndim;
  const double* src = Y;
  for (int a = 0, k = 1; a < d; ++a, ++k) {
    double* dst = ((d - k) % 2 == 0) ? U : S;
    axis_pass(h, a, false, src, dst, ntc);
    src = dst;
  }
}

void check_solvable(const stkg_heat& h) {
  if (h.singular) {
    char buf[160];
    snprintf(buf, sizeof buf, "solve_projected_heat: singular row system at lambda = %f",
             h.singular_lambda);
    throw Error(STKG_SINGULARITY, buf);
  }
}

template <int NDIM>
int64_t apply_tiles(const stkg_heat& h) {
  using T = ApplyTile<NDIM>;
  return ceil_div(h.n[0], T::BX) * ceil_div(h.n[1], T::BY) * ceil_div(h.n[2], T::BZ);
}

// 2D / 3D: tiles x time chunks of heat_apply2d_kernel / heat_apply3d_kernel (STKG_K1_XMARCH=0:
// the generic kernel)
bool use_apply_xmarch() {
  static const bool on = [] {
    const char* e = std::getenv("STKG_K1_XMARCH");
    return !(e && e[0] == '0');
  }();
  return on;
}
int64_t apply2d_blocks(const stkg_heat& h, int64_t nt) {
  return ceil_div(h.n[0], Apply2D::BX) * ceil_div(h.n[1], Apply2D::BY) *
         std::max<int64_t>(1, ceil_div(nt, Apply2D::kChunk));
}

int64_t apply3d_blocks(const stkg_heat& h, int64_t nt) {
  return ceil_div(h.n[0], Apply3D::BX) * ceil_div(h.n[1], Apply3D::BY) *
         ceil_div(h.n[2], Apply3D::BZ) * std::max<int64_t>(1, ceil_div(nt, Apply3D::kChunk));
}

int64_t apply_blocks(const stkg_heat& h) {
  if (h.ndim == 2 && use_apply_xmarch()) return apply2d_blocks(h, h.nt);
  if (h.ndim == 3 && use_apply_xmarch()) return apply3d_blocks(h, h.nt);
  return h.ndim == 1 ? apply_tiles<1>(h) : (h.ndim == 2 ? apply_tiles<2>(h) : apply_tiles<3>(h));
}

template <int NDIM, bool RES>
void launch_apply(stkg_heat& h, const double* U, const double* F, double* out, int64_t nt,
                  const double* dd, const double* ds, const double* cd, const double* cs) {
  const unsigned blocks = static_cast<unsigned>(apply_tiles<NDIM>(h));
  Tri m[3], a[3];
  for (int i = 0; i < 3; ++i) {
    m[i] = Tri{h.m_diag[i].p, h.m_off[i].p};
    a[i] = Tri{h.a_diag[i].p, h.a_off[i].p};
  }
  if constexpr (NDIM == 2) {
    if (use_apply_xmarch()) {
      static const bool configured2 = [] {
        STKG_CUDA_CHECK(cudaFuncSetAttribute(heat_apply2d_kernel<RES>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(apply2d_smem<RES>())));
        return true;
      }();
      (void)configured2;
      heat_apply2d_kernel<RES><<<static_cast<unsigned>(apply2d_blocks(h, nt)), 256,
                                 apply2d_smem<RES>(), h.stream>>>(
          U, F, out, h.n[0], h.n[1], nt, m[0], m[1], a[0], a[1], dd, ds, cd, cs, h.partials.p);
      STKG_CUDA_CHECK(cudaGetLastError());
      return;
    }
  }
  if constexpr (NDIM == 3) {
    if (use_apply_xmarch()) {
      static const bool configured3 = [] {
        STKG_CUDA_CHECK(cudaFuncSetAttribute(heat_apply3d_kernel<RES>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(apply3d_smem<RES>())));
        return true;
      }();
      (void)configured3;
      heat_apply3d_kernel<RES><<<static_cast<unsigned>(apply3d_blocks(h, nt)), 256,
                                 apply3d_smem<RES>(), h.stream>>>(
          U, F, out, h.n[0], h.n[1], h.n[2], nt, m[0], m[1], m[2], a[0], a[1], a[2], dd, ds,
          cd, cs, h.partials.p);
      STKG_CUDA_CHECK(cudaGetLastError());
      return;
    }
  }
  using SM = ApplySmem<NDIM, RES>;
  static const bool configured = [] {
    STKG_CUDA_CHECK(cudaFuncSetAttribute(heat_apply_kernel<NDIM, RES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(SM::kBytes)));
    return true;
  }();
  (void)configured;
  heat_apply_kernel<NDIM, RES><<<blocks, 256, SM::kBytes, h.stream>>>(
      U, F, out, h.n[0], h.n[1], h.n[2], nt, m[0], m[1], m[2], a[0], a[1], a[2], dd, ds, cd, cs,
      h.partials.p);
  STKG_CUDA_CHECK(cudaGetLastError());
}

template <bool RES>
void dispatch_apply(stkg_heat& h, const double* U, const double* F, double* out, int64_t nt,
                    const double* dd, const double* ds, const double* cd, const double* cs) {
  if (h.ndim == 1) launch_apply<1, RES>(h, U, F, out, nt, dd, ds, cd, cs);
  else if (h.ndim == 2) launch_apply<2, RES>(h, U, F, out, nt, dd, ds, cd, cs);
  else launch_apply<3, RES>(h, U, F, out, nt, dd, ds, cd, cs);
}

template <bool RES>
void dispatch_apply(stkg_heat& h, const double* U, const double* F, double* out) {
  dispatch_apply<RES>(h, U, F, out, h.nt, h.d_diag.p, h.d_sup.p, h.c_diag.p, h.c_sup.p);
}

}  // namespace

namespace stkg {
void apply_with_time(stkg_heat& h, const double* U, double* out, int64_t nt, const double* dd,
                     const double* ds, const double* cd, const double* cs) {
  STKG_REQUIRE(h.has_operator, STKG_ARGUMENT, "apply: plan was created without the spatial factors");
  dispatch_apply<false>(h, U, nullptr, out, nt, dd, ds, cd, cs);
}
}  // namespace stkg

namespace {
// sin(pi r / N) and cos(pi r / N) for integers r, N with exact range reduction
double sinpi_ratio_h(int64_t r, int64_t N) {
  int64_t m = r % (2 * N);
  if (m < 0) m += 2 * N;
  double sign = 1.0;
  if (m >= N) {
    m -= N;
    sign = -1.0;
  }
  if (2 * m > N) m = N - m;
  return sign * std::sin(M_PI * static_cast<double>(m) / static_cast<double>(N));
}
double cospi_ratio(int64_t r, int64_t N) { return sinpi_ratio_h(2 * r + N, 2 * N); }

std::vector<double> transpose(const double* X, int64_t n) {
  std::vector<double> t(static_cast<size_t>(n * n));
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) t[i * n + j] = X[j * n + i];
  return t;
}

}  // namespace

namespace {
// STKG_TRIDIAG=0 keeps the transform-based fused pass (heat_fused.cuh).
bool tridiag_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("STKG_TRIDIAG");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

// Line-solve axis-0 pass (heat_tridiag.cuh): uniform time grid, axis 0 a uniform P1 axis whose
// pencil the caller's eigenvalues confirm (lambda_k mu_k = a_d + 2 a_o cos(pi k / N) with the
// P1 stencils M_0 = (h/6) tridiag(1, 4, 1), A_0 = (1/h) tridiag(-1, 2, -1)), every column's
// T_c positive definite.  Otherwise the plan keeps the transform-based pass.
void setup_tridiag(stkg_heat& h, const double* lam0, double hh) {
  h.tri_ok = false;
  if (!tridiag_enabled() || h.pitch <= 0 || h.lam_col.p == nullptr) return;
  // non-uniform time grids: the TMA variant recomputes its per-column constants every step
  // (STKG_TRI_NONUNIFORM=0 keeps the fused transform pass for them); the LDL^T variant's pivot
  // table is per plan
  static const bool nonuni_on = [] {
    const char* e = std::getenv("STKG_TRI_NONUNIFORM");
    return !(e && std::atoi(e) == 0);
  }();
  if (!h.uniform_time && (tri_variant() == 0 || !nonuni_on)) return;
  const int64_t n0 = h.n[0], N = n0 + 1;
  if (tri_tile_cols(n0) == 0) return;
  const double md = 2.0 * hh / 3.0, mo = hh / 6.0, ad = 2.0 / hh, ao = -1.0 / hh;
  for (int64_t k = 1; k <= n0; ++k) {
    const double ck = cospi_ratio(k, N);
    const double alpha = lam0[k - 1] * (md + 2.0 * mo * ck), want = ad + 2.0 * ao * ck;
    if (!(std::fabs(alpha - want) <= 1e-9 * ad)) return;
  }
  int64_t inner = h.pitch;
  for (int b = 1; b + 1 < h.ndim; ++b) inner *= h.n[b];
  if (inner % tri_tile_cols(n0) != 0) return;
  h.tri_md = md, h.tri_mo = mo, h.tri_ad = ad, h.tri_ao = ao;
  // every column's T_c = tridiag(a, b, a) must have a positive symbol (b > 2|a|), a moderate
  // condition number and a decay q = |a| / w with q^N below 1 (the image sums divide by
  // 1 - q^{2N})
  std::vector<double> lc(static_cast<size_t>(inner));
  STKG_CUDA_CHECK(cudaMemcpyAsync(lc.data(), h.lam_col.p, inner * sizeof(double),
                                  cudaMemcpyDeviceToHost, h.stream));
  STKG_CUDA_CHECK(cudaStreamSynchronize(h.stream));
  // (the symbol is affine in lambda_c, so per step only the extreme columns need the test)
  double lmin = lc[0], lmax = lc[0];
  for (int64_t c = 1; c < inner; ++c) lmin = std::min(lmin, lc[c]), lmax = std::max(lmax, lc[c]);
  const int64_t steps = h.uniform_time ? 1 : h.nt;
  for (int64_t l = 0; l < steps; ++l) {
    const double dd = h.d_diag_h[l], cd = h.c_diag_h[l];
    for (const double lam : {lmin, lmax}) {
      const double p = dd + lam * cd;
      const double b = p * md + cd * ad;
      const double bp = p * (md + 2.0 * mo) + cd * (ad + 2.0 * ao);
      const double bm = p * (md - 2.0 * mo) + cd * (ad - 2.0 * ao);
      if (!(b > 0.0 && bp > 0.0 && bm > 0.0)) return;
    }
    // q = |a| / w is largest where b / |a| is smallest: test every column on uniform grids,
    // the extreme columns and a sample in between otherwise
    const int64_t stride = h.uniform_time ? 1 : std::max<int64_t>(1, inner / 64);
    for (int64_t c = 0; c < inner; c += stride) {
      const double p = dd + lc[c] * cd;
      const double a = p * mo + cd * ao, b = p * md + cd * ad;
      const double bp = p * (md + 2.0 * mo) + cd * (ad + 2.0 * ao);
      const double bm = p * (md - 2.0 * mo) + cd * (ad - 2.0 * ao);
      if (!(b > 0.0 && bp > 0.0 && bm > 0.0)) return;
      // a tridiagonal line solve loses cond(T_c) = max(b + 2a, b - 2a) / min(...) ulps (the
      // modal recurrence divides mode by mode and loses none): plans with very large time
      // steps against h^2 (measured 5.5e-12 against the DMMA backend at cond 1e6) keep the
      // transform pass; cfg3 has cond 2e3, cfg5 1.3e2
      if (!(std::max(bp, bm) <= 1e5 * std::min(bp, bm))) return;
      const double q = std::fabs(a) / (0.5 * (b + std::sqrt(bp * bm)));
      if (!(std::pow(q, static_cast<double>(N)) < 0.9)) return;
    }
  }
  h.tri_ok = true;
  if (tri_variant() != 0) return;
  // the cp.async LDL^T variant keeps a table of reciprocal pivots
  h.tri_iw.alloc(static_cast<size_t>(N * inner));
  int* bad = nullptr;
  STKG_CUDA_CHECK(cudaMalloc(&bad, sizeof(int)));
  STKG_CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), h.stream));
  tri_factor_kernel<<<static_cast<unsigned>(ceil_div(inner, 128)), 128, 0, h.stream>>>(
      h.tri_iw.p, inner, static_cast<int>(n0), h.lam_col.p, h.d_diag_h[0], h.c_diag_h[0], md, mo,
      ad, ao, bad);
  int hb = 1;
  cudaError_t e1 = cudaGetLastError();
  cudaError_t e2 = cudaMemcpyAsync(&hb, bad, sizeof hb, cudaMemcpyDeviceToHost, h.stream);
  cudaError_t e3 = cudaStreamSynchronize(h.stream);
  cudaFree(bad);
  STKG_CUDA_CHECK(e1);
  STKG_CUDA_CHECK(e2);
  STKG_CUDA_CHECK(e3);
  h.tri_ok = hb == 0;
  if (!h.tri_ok) h.tri_iw.release();
}
}  // namespace

// ------------------------------------------------------------------------ C ABI -----
extern "C" {

int stkg_fill_uniform(double* dst, int64_t count, uint64_t seed, uint64_t stream,
                      int64_t index_offset, void* cuda_stream) {
  return guarded([&] {
    STKG_REQUIRE(count >= 0 && (dst || count == 0), STKG_ARGUMENT, "fill_uniform: bad args");
    if (count == 0) return;
    fill_uniform_kernel<<<num_sms() * 8, 256, 0, static_cast<cudaStream_t>(cuda_stream)>>>(
        dst, count, seed, stream, index_offset);
    STKG_CUDA_CHECK(cudaGetLastError());
  });
}

int stkg_heat_create(stkg_heat** out, const stkg_heat_desc* desc, void* cuda_stream) {
  return guarded([&] {
    STKG_REQUIRE(out && desc, STKG_ARGUMENT, "stkg_heat_create: null argument");
    *out = nullptr;
    STKG_REQUIRE(desc->ndim >= 1 && desc->ndim <= 3, STKG_ARGUMENT,
                 "stkg_heat_create: ndim must be 1, 2 or 3");
    STKG_REQUIRE(desc->nt >= 1, STKG_ARGUMENT, "stkg_heat_create: nt must be >= 1");
    auto h = std::make_unique<stkg_heat>();
    h->ndim = desc->ndim;
    h->nt = desc->nt;
    h->nx = 1;
    h->transform = desc->transform;
    STKG_REQUIRE(h->transform == STKG_TRANSFORM_DENSE || h->transform == STKG_TRANSFORM_P1_DST,
                 STKG_ARGUMENT, "stkg_heat_create: unknown transform");
    const bool dst_mode = h->transform == STKG_TRANSFORM_P1_DST;
    for (int a = 0; a < h->ndim; ++a) {
      STKG_REQUIRE(desc->n[a] >= 1, STKG_ARGUMENT, "stkg_heat_create: n must be >= 1");
      STKG_REQUIRE((dst_mode || desc->X[a]) && desc->lambdas[a], STKG_ARGUMENT,
                   "stkg_heat_create: missing EigPair for an axis");
      if (dst_mode) {
        const int64_t N = desc->n[a] + 1;
        STKG_REQUIRE(N >= 16 && N <= 2048 && (N & (N - 1)) == 0, STKG_ARGUMENT,
                     "P1_DST transform: n + 1 must be a power of two in [16, 2048]");
        STKG_REQUIRE(desc->p1_h[a] > 0.0, STKG_ARGUMENT, "P1_DST transform: p1_h must be > 0");
      }
      h->n[a] = desc->n[a];
      h->nx *= desc->n[a];
    }
    STKG_REQUIRE(desc->d_diag && desc->c_diag && (desc->nt == 1 || (desc->d_sup && desc->c_sup)),
                 STKG_ARGUMENT, "stkg_heat_create: missing temporal bidiagonals");
    h->stream = static_cast<cudaStream_t>(cuda_stream);
    cudaStream_t s = h->stream;
    for (int a = 0; a < h->ndim; ++a) {
      const int64_t na = h->n[a];
      h->lam[a].alloc(na);
      h->lam[a].upload(desc->lambdas[a], na, s);
      h->lam_h[a].assign(desc->lambdas[a], desc->lambdas[a] + na);
      if (dst_mode) {
        // 1/mu_k with mu_k = (h/3)(2 + cos(pi k/N)), k = 1..n (the M_h eigenvalues), and the
        // 2N-th roots of unity, both with exact integer argument reduction.
        const int64_t N = na + 1, L = 2 * N;
        std::vector<double> w(na), tw(2 * L);
        const double hh = desc->p1_h[a];
        for (int64_t k = 1; k <= na; ++k) w[k - 1] = 1.0 / ((hh / 3.0) * (2.0 + cospi_ratio(k, N)));
        for (int64_t m = 0; m < L; ++m) {
          tw[2 * m] = cospi_ratio(2 * m, L);        // cos(2 pi m / L)
          tw[2 * m + 1] = -sinpi_ratio_h(2 * m, L);  // -sin(2 pi m / L)
        }
        h->inv_mu[a].alloc(na);
        h->inv_mu[a].upload(w.data(), na, s);
        h->twiddle[a].alloc(2 * L);
        h->twiddle[a].upload(tw.data(), 2 * L, s);
      } else {
        h->X[a].alloc(na * na);
        h->X[a].upload(desc->X[a], na * na, s);
        auto t = transpose(desc->X[a], na);
        h->XT[a].alloc(na * na);
        h->XT[a].upload(t.data(), na * na, s);
      }
      STKG_CUDA_CHECK(cudaStreamSynchronize(s));  // host temporaries die here
    }
    const int64_t nt = h->nt;
    {  // uniform time grid: every step has the same bidiagonal coefficients
      bool u = true;
      for (int64_t l = 1; l < nt; ++l)
        u = u && desc->d_diag[l] == desc->d_diag[0] && desc->c_diag[l] == desc->c_diag[0];
      for (int64_t l = 1; l + 1 < nt; ++l)
        u = u && desc->d_sup[l] == desc->d_sup[0] && desc->c_sup[l] == desc->c_sup[0];
      h->uniform_time = u;
    }
    h->d_diag_h.assign(desc->d_diag, desc->d_diag + nt);
    h->c_diag_h.assign(desc->c_diag, desc->c_diag + nt);
    if (nt > 1) {
      h->d_sup_h.assign(desc->d_sup, desc->d_sup + nt - 1);
      h->c_sup_h.assign(desc->c_sup, desc->c_sup + nt - 1);
    }
    h->d_diag.alloc(nt);
    h->d_diag.upload(desc->d_diag, nt, s);
    h->c_diag.alloc(nt);
    h->c_diag.upload(desc->c_diag, nt, s);
    h->d_sup.alloc(std::max<int64_t>(nt - 1, 1));
    h->c_sup.alloc(std::max<int64_t>(nt - 1, 1));
    if (nt > 1) {
      h->d_sup.upload(desc->d_sup, nt - 1, s);
      h->c_sup.upload(desc->c_sup, nt - 1, s);
    }
    bool op = true;
    for (int a = 0; a < h->ndim; ++a)
      op = op && desc->m_diag[a] && desc->a_diag[a] &&
           (h->n[a] == 1 || (desc->m_off[a] && desc->a_off[a]));
    h->has_operator = op;
    for (int a = 0; a < 3; ++a) {
      // unused axes get the 1x1 identity/zero factors so the stencil code is uniform
      const int64_t na = a < h->ndim ? h->n[a] : 1;
      h->m_diag[a].alloc(na);
      h->a_diag[a].alloc(na);
      h->m_off[a].alloc(std::max<int64_t>(na - 1, 1));
      h->a_off[a].alloc(std::max<int64_t>(na - 1, 1));
      if (a < h->ndim && op) {
        h->m_diag_h[a].assign(desc->m_diag[a], desc->m_diag[a] + na);
        h->a_diag_h[a].assign(desc->a_diag[a], desc->a_diag[a] + na);
        if (na > 1) {
          h->m_off_h[a].assign(desc->m_off[a], desc->m_off[a] + na - 1);
          h->a_off_h[a].assign(desc->a_off[a], desc->a_off[a] + na - 1);
        }
        h->m_diag[a].upload(desc->m_diag[a], na, s);
        h->a_diag[a].upload(desc->a_diag[a], na, s);
        if (na > 1) {
          h->m_off[a].upload(desc->m_off[a], na - 1, s);
          h->a_off[a].upload(desc->a_off[a], na - 1, s);
        }
      } else if (a >= h->ndim) {
        const double one = 1.0, zero = 0.0;
        STKG_CUDA_CHECK(cudaMemcpyAsync(h->m_diag[a].p, &one, 8, cudaMemcpyHostToDevice, s));
        STKG_CUDA_CHECK(cudaMemcpyAsync(h->a_diag[a].p, &zero, 8, cudaMemcpyHostToDevice, s));
        STKG_CUDA_CHECK(cudaStreamSynchronize(s));
      }
    }
    // padded internal layout of the device solve (run_chunk_padded): P1_DST 2D/3D plans whose
    // axes all have half-length kernels; STKG_PAD=0 keeps the unpadded passes
    if (dst_mode && h->ndim >= 2 && use_dst_half() && padded_layout_enabled()) {
      bool ok = true;
      for (int a = 0; a < h->ndim; ++a) {
        const int64_t N = h->n[a] + 1;
        ok = ok && N >= 16 && N <= 1024 && (N & (N - 1)) == 0;
      }
      if (ok) {
        const int last = h->ndim - 1;
        const int64_t nl = h->n[last];
        h->pitch = nl + 1;
        std::vector<double> lp(desc->lambdas[last], desc->lambdas[last] + nl);
        lp.push_back(0.0);
        h->lam_pad.alloc(nl + 1);
        h->lam_pad.upload(lp.data(), nl + 1, s);
        std::vector<double> wp(nl + 1, 0.0);
        STKG_CUDA_CHECK(cudaMemcpyAsync(wp.data(), h->inv_mu[last].p, nl * sizeof(double),
                                        cudaMemcpyDeviceToHost, s));
        STKG_CUDA_CHECK(cudaStreamSynchronize(s));
        h->inv_mu_pad.alloc(nl + 1);
        h->inv_mu_pad.upload(wp.data(), nl + 1, s);
        // per-column eigenvalue sums and weight products of the axes faster than axis 0
        // (the fused axis-0 pass, heat_fused.cuh)
        if (h->ndim == 2) {
          h->lam_col.alloc(nl + 1);
          h->lam_col.upload(lp.data(), nl + 1, s);
          h->w_col.alloc(nl + 1);
          h->w_col.upload(wp.data(), nl + 1, s);
        } else {
          const int64_t n1 = h->n[1];
          std::vector<double> w1(n1);
          STKG_CUDA_CHECK(cudaMemcpyAsync(w1.data(), h->inv_mu[1].p, n1 * sizeof(double),
                                          cudaMemcpyDeviceToHost, s));
          STKG_CUDA_CHECK(cudaStreamSynchronize(s));
          std::vector<double> lc(n1 * (nl + 1)), wc(n1 * (nl + 1));
          for (int64_t iy = 0; iy < n1; ++iy)
            for (int64_t iz = 0; iz <= nl; ++iz) {
              lc[iy * (nl + 1) + iz] = desc->lambdas[1][iy] + lp[iz];
              wc[iy * (nl + 1) + iz] = w1[iy] * wp[iz];
            }
          h->lam_col.alloc(lc.size());
          h->lam_col.upload(lc.data(), lc.size(), s);
          h->w_col.alloc(wc.size());
          h->w_col.upload(wc.data(), wc.size(), s);
        }
        STKG_CUDA_CHECK(cudaStreamSynchronize(s));
        setup_tridiag(*h, desc->lambdas[0], desc->p1_h[0]);
      }
    }
    h->carry.alloc(h->pitch > 0 ? padded_nx(*h) : h->nx);
    h->partials.alloc(2 * apply_blocks(*h));
    h->scalars.alloc(4);
    STKG_CUDA_CHECK(cudaMallocHost(&h->pinned, 4 * sizeof(double)));
    h->time_chunk = desc->time_chunk;

    // one-time pivot check (stk/sylvester.hpp:133-135)
    unsigned long long* bad = nullptr;
    STKG_CUDA_CHECK(cudaMalloc(&bad, sizeof(unsigned long long)));
    STKG_CUDA_CHECK(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
    heat_pivot_check_kernel<<<static_cast<unsigned>(ceil_div(h->nx, 256)), 256, 0, s>>>(
        h->nx, h->nt, mode_lambda(*h), h->d_diag.p, h->c_diag.p, bad);
    STKG_CUDA_CHECK(cudaGetLastError());
    unsigned long long hb = 0;
    STKG_CUDA_CHECK(cudaMemcpyAsync(&hb, bad, sizeof hb, cudaMemcpyDeviceToHost, s));
    STKG_CUDA_CHECK(cudaStreamSynchronize(s));
    cudaFree(bad);
    if (hb != ~0ull) {
      h->singular = 1;
      const int64_t i = static_cast<int64_t>(hb % static_cast<unsigned long long>(h->nx));
      h->singular_step = static_cast<int64_t>(hb / static_cast<unsigned long long>(h->nx));
      // reconstruct lambda_i on the host for the message
      std::vector<double> li(1);
      int64_t idx[3] = {i, 0, 0};
      if (h->ndim == 2) idx[0] = i / h->n[1], idx[1] = i % h->n[1];
      if (h->ndim == 3) idx[2] = i % h->n[2], idx[1] = (i / h->n[2]) % h->n[1],
                        idx[0] = i / (h->n[1] * h->n[2]);
      double lam = 0.0;
      for (int a = 0; a < h->ndim; ++a) lam += desc->lambdas[a][idx[a]];
      h->singular_lambda = lam;
    }
    *out = h.release();
  });
}

int stkg_heat_destroy(stkg_heat* h) {
  return guarded([&] {
    if (!h) return;
    if (h->stream) cudaStreamSynchronize(h->stream);
    else cudaDeviceSynchronize();
    if (h->pinned) cudaFreeHost(h->pinned);
    if (h->rk_pin) cudaFreeHost(h->rk_pin);
    for (int c = 0; c < 2; ++c)
      for (auto e : h->prof_ev[c]) cudaEventDestroy(e);  // profiling left enabled
    for (int b = 0; b < 2; ++b) {
      if (h->ev_h2d[b]) cudaEventDestroy(h->ev_h2d[b]);
      if (h->ev_comp[b]) cudaEventDestroy(h->ev_comp[b]);
      if (h->ev_d2h[b]) cudaEventDestroy(h->ev_d2h[b]);
    }
    if (h->s_h2d) cudaStreamDestroy(h->s_h2d);
    if (h->s_hi) cudaStreamSynchronize(h->s_hi), cudaStreamDestroy(h->s_hi);
    if (h->s_lo) cudaStreamSynchronize(h->s_lo), cudaStreamDestroy(h->s_lo);
    for (auto e : h->ov_ev) cudaEventDestroy(e);
    if (h->tickets) cudaFree(h->tickets);
    if (h->s_d2h) cudaStreamDestroy(h->s_d2h);
    delete h;
  });
}

int stkg_heat_schedule(const stkg_heat* h) {
  if (!h || h->pitch <= 0) return STKG_SCHEDULE_SEPARATE;
  int64_t inner0 = h->pitch;
  for (int b = 1; b + 1 < h->ndim; ++b) inner0 *= h->n[b];
  try {
    if (!use_fused_axis0(*h, inner0)) return STKG_SCHEDULE_SEPARATE;
    return use_tridiag(*h, inner0) ? STKG_SCHEDULE_LINE_SOLVE : STKG_SCHEDULE_FUSED_DST;
  } catch (...) {
    return STKG_SCHEDULE_SEPARATE;
  }
}

int64_t stkg_heat_workspace_bytes(const stkg_heat* h) {
  if (!h) return 0;
  int64_t b = 0;
  const DevBuf* bufs[] = {&h->scratch, &h->lfac, &h->carry, &h->partials, &h->pf[0], &h->pf[1],
                          &h->pu[0],   &h->pu[1], &h->ps};
  for (auto* x : bufs) b += static_cast<int64_t>(x->n) * 8;
  for (int a = 0; a < h->ndim; ++a)
    b += static_cast<int64_t>(2 * h->X[a].n + h->lam[a].n + h->inv_mu[a].n + h->twiddle[a].n) * 8;
  return b;
}

int stkg_heat_solve(stkg_heat* h, const double* F, double* U) {
  return guarded([&] {
    STKG_REQUIRE(h && F && U, STKG_ARGUMENT, "stkg_heat_solve: null argument");
    {  // no overlap at all: the overlapped 2D schedule reads F and writes U concurrently
      const int64_t N = h->nx * h->nt;
      const auto f0 = reinterpret_cast<uintptr_t>(F), u0 = reinterpret_cast<uintptr_t>(U);
      const auto bytes = static_cast<uintptr_t>(N) * sizeof(double);
      STKG_REQUIRE(f0 + bytes <= u0 || u0 + bytes <= f0, STKG_ARGUMENT,
                   "stkg_heat_solve: U may not alias F");
    }
    check_solvable(*h);
    solve_range(*h, F, U, 0, h->nt);
  });
}

int stkg_heat_solve_factored(stkg_heat* h, int64_t rank, const double* L, const double* R,
                             double* U) {
  return guarded([&] {
    STKG_REQUIRE(h && L && R && U, STKG_ARGUMENT, "stkg_heat_solve_factored: null argument");
    STKG_REQUIRE(rank >= 1 && rank <= kMaxFactorRank, STKG_ARGUMENT,
                 "stkg_heat_solve_factored: rank must be in [1, 16]");
    check_solvable(*h);
    if (h->scratch.n < static_cast<size_t>(h->nx * h->nt)) h->scratch.alloc(h->nx * h->nt);
    if (h->lfac.n < static_cast<size_t>(2 * h->nx * rank)) h->lfac.alloc(2 * h->nx * rank);
    // forward transforms of the rank columns of L (treated as `rank` time slices)
    double* t0 = h->lfac.p;
    double* t1 = h->lfac.p + h->nx * rank;
    const double* src = L;
    for (int a = h->ndim - 1, k = 1; a >= 0; --a, ++k) {
      double* dst = ((h->ndim - k) % 2 == 0) ? t0 : t1;
      axis_pass(*h, a, true, src, dst, rank);
      src = dst;
    }
    const int rp = factor_rp(rank);
    if (h->rt.n < static_cast<size_t>(h->nt * rp)) h->rt.alloc(h->nt * rp);
    factor_transpose_kernel<<<static_cast<unsigned>(ceil_div(h->nt * rp, 256)), 256, 0, h->stream>>>(
        R, rank, h->nt, rp, h->rt.p);
    STKG_CUDA_CHECK(cudaGetLastError());
    const double* Rt = h->rt.p;
    if (h->pitch > 0) {  // padded layout: Y~ in the scratch, inverse passes as run_chunk_padded
      const int64_t nxp = padded_nx(*h), last = h->ndim - 1;
      if (h->scratch.n < static_cast<size_t>(nxp * h->nt)) h->scratch.alloc(nxp * h->nt);
      double* S = h->scratch.p;
      {
        ProfScope ps(*h, 1);
        launch_factored(h->uniform_time, rp)<<<static_cast<unsigned>(ceil_div(nxp, 256)), 256, 0, h->stream>>>(
            src, Rt, static_cast<int>(rank), S, nxp, h->nt, mode_lambda_padded(*h),
            mode_weight_padded(*h), h->d_diag.p, h->d_sup.p, h->c_diag.p, h->c_sup.p, h->pitch,
            h->n[last]);
        STKG_CUDA_CHECK(cudaGetLastError());
      }
      inverse_passes_padded(*h, S, U, h->nt);
      return;
    }
    // the recurrence writes Y~ where the first inverse pass reads it
    double* Y = (h->ndim % 2 == 0) ? U : h->scratch.p;
    {
      ProfScope ps(*h, 1);
      launch_factored(h->uniform_time, rp)<<<static_cast<unsigned>(ceil_div(h->nx, 256)), 256, 0, h->stream>>>(
          src, Rt, static_cast<int>(rank), Y, h->nx, h->nt, mode_lambda(*h), mode_weight(*h), h->d_diag.p,
          h->d_sup.p, h->c_diag.p, h->c_sup.p, 0, 0);
      STKG_CUDA_CHECK(cudaGetLastError());
    }
    inverse_passes(*h, Y, U, h->scratch.p, h->nt);
  });
}

int stkg_heat_solve_host(stkg_heat* h, const double* F_host, double* U_host) {
  return guarded([&] {
    STKG_REQUIRE(h && F_host && U_host, STKG_ARGUMENT, "stkg_heat_solve_host: null argument");
    check_solvable(*h);
    int64_t tc = h->time_chunk;
    if (tc <= 0) tc = std::max<int64_t>(1, (int64_t(256) << 20) / (h->nx * 8));
    tc = std::min(tc, h->nt);
    const int64_t chunk_elems = h->nx * tc;
    if (h->pf[0].n < static_cast<size_t>(chunk_elems)) {
      STKG_CUDA_CHECK(cudaStreamSynchronize(h->stream));
      for (int b = 0; b < 2; ++b) {
        h->pf[b].alloc(chunk_elems);
        h->pu[b].alloc(chunk_elems);
      }
    }
    if (!h->s_h2d) {
      STKG_CUDA_CHECK(cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking));
      STKG_CUDA_CHECK(cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
      for (int b = 0; b < 2; ++b) {
        STKG_CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_h2d[b], cudaEventDisableTiming));
        STKG_CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_comp[b], cudaEventDisableTiming));
        STKG_CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_d2h[b], cudaEventDisableTiming));
      }
    }
    const int64_t nchunks = ceil_div(h->nt, tc);
    for (int64_t c = 0; c < nchunks; ++c) {
      const int b = static_cast<int>(c & 1);
      const int64_t l0 = c * tc, ntc = std::min(tc, h->nt - l0);
      const size_t bytes = static_cast<size_t>(h->nx * ntc) * sizeof(double);
      if (c >= 2) STKG_CUDA_CHECK(cudaStreamWaitEvent(h->s_h2d, h->ev_comp[b], 0));
      STKG_CUDA_CHECK(cudaMemcpyAsync(h->pf[b].p, F_host + l0 * h->nx, bytes,
                                      cudaMemcpyHostToDevice, h->s_h2d));
      STKG_CUDA_CHECK(cudaEventRecord(h->ev_h2d[b], h->s_h2d));
      STKG_CUDA_CHECK(cudaStreamWaitEvent(h->stream, h->ev_h2d[b], 0));
      if (c >= 2) STKG_CUDA_CHECK(cudaStreamWaitEvent(h->stream, h->ev_d2h[b], 0));
      solve_range(*h, h->pf[b].p, h->pu[b].p, l0, ntc);
      STKG_CUDA_CHECK(cudaEventRecord(h->ev_comp[b], h->stream));
      STKG_CUDA_CHECK(cudaStreamWaitEvent(h->s_d2h, h->ev_comp[b], 0));
      STKG_CUDA_CHECK(cudaMemcpyAsync(U_host + l0 * h->nx, h->pu[b].p, bytes,
                                      cudaMemcpyDeviceToHost, h->s_d2h));
      STKG_CUDA_CHECK(cudaEventRecord(h->ev_d2h[b], h->s_d2h));
    }
    STKG_CUDA_CHECK(cudaStreamSynchronize(h->s_d2h));
    STKG_CUDA_CHECK(cudaStreamSynchronize(h->stream));
  });
}

int stkg_heat_profile(stkg_heat* h, int enable, double* ms_out, int64_t* launches_out) {
  return guarded([&] {
    STKG_REQUIRE(h, STKG_ARGUMENT, "stkg_heat_profile: null plan");
    auto drop = [&] {
      for (int c = 0; c < 2; ++c) {
        for (auto e : h->prof_ev[c]) cudaEventDestroy(e);
        h->prof_ev[c].clear();
      }
    };
    if (enable) {
      drop();
      h->prof_launches[0] = h->prof_launches[1] = 0;
      h->prof_on = true;
      return;
    }
    h->prof_on = false;
    STKG_CUDA_CHECK(cudaStreamSynchronize(h->stream));
    for (int c = 0; c < 2; ++c) {
      double ms = 0.0;
      for (size_t i = 0; i + 1 < h->prof_ev[c].size(); i += 2) {
        float t = 0.f;
        STKG_CUDA_CHECK(cudaEventElapsedTime(&t, h->prof_ev[c][i], h->prof_ev[c][i + 1]));
        ms += t;
      }
      if (ms_out) ms_out[c] = ms;
      if (launches_out) launches_out[c] = h->prof_launches[c];
    }
    drop();
  });
}

int stkg_heat_apply(stkg_heat* h, const double* U, double* out) {
  return guarded([&] {
    STKG_REQUIRE(h && U && out, STKG_ARGUMENT, "stkg_heat_apply: null argument");
    STKG_REQUIRE(h->has_operator, STKG_ARGUMENT,
                 "stkg_heat_apply: plan was created without the spatial factors");
    STKG_REQUIRE(U != out, STKG_ARGUMENT, "stkg_heat_apply: out may not alias U");
    dispatch_apply<false>(*h, U, nullptr, out);
  });
}

int stkg_heat_residual(stkg_heat* h, const double* U, const double* F, double* relres,
                       double* fnorm) {
  return guarded([&] {
    STKG_REQUIRE(h && U && F, STKG_ARGUMENT, "stkg_heat_residual: null argument");
    STKG_REQUIRE(h->has_operator, STKG_ARGUMENT,
                 "stkg_heat_residual: plan was created without the spatial factors");
    dispatch_apply<true>(*h, U, F, nullptr);
    sum_pairs_kernel<<<1, 256, 0, h->stream>>>(h->partials.p, apply_blocks(*h), h->scalars.p);
    STKG_CUDA_CHECK(cudaGetLastError());
    STKG_CUDA_CHECK(cudaMemcpyAsync(h->pinned, h->scalars.p, 2 * sizeof(double),
                                    cudaMemcpyDeviceToHost, h->stream));
    STKG_CUDA_CHECK(cudaStreamSynchronize(h->stream));
    const double rn = std::sqrt(h->pinned[0]), fn = std::sqrt(h->pinned[1]);
    if (fnorm) *fnorm = fn;
    if (relres) *relres = fn > 0 ? rn / fn : rn;
  });
}

}  // extern "C"
