// FP64 tensor-core GEMM for sm_100a (K2 of SURVEY §2.1): C_b = A_b * B_b, column-major,
// arbitrary M/N/K and leading dimensions (8-byte aligned operands are enough: the heat
// slices of U have leading dimension n = 1023).
//
// sm_100a has no tcgen05 FP64 kind (ptxas rejects kind::f64), so the FP64 tensor path is
// the warp-level mma.sync.m16n8k4.f64, which lowers to DMMA.8x8x4.  Measured on B200:
// DMMA 37.1 TFLOP/s vs DFMA 34.2 TFLOP/s (profiles/r01_fp64_peak.txt), so the transforms
// run on DMMA.  Operands are staged by a multi-stage cp.async pipeline (8-byte granules,
// zero-filled at the matrix edges), fragments are read from padded, bank-conflict-free
// shared memory tiles.
//
// These GEMMs are the basis transforms of solve_projected_heat_with
// (stk/sylvester.hpp:126 `eig.X.transpose() * g`, :141 `eig.X * yt`) in tensor form, and
// the four products of TwoTermPrecond::solve (stk/sylvester.hpp:171,175).
#pragma once

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace stkg {

struct GemmProblem {
  int64_t M = 0, N = 0, K = 0;
  int64_t batch = 1;
  const double* A = nullptr;  // M x K, column-major
  int64_t lda = 0, strideA = 0;
  const double* B = nullptr;  // K x N, column-major
  int64_t ldb = 0, strideB = 0;
  double* C = nullptr;        // M x N, column-major
  int64_t ldc = 0, strideC = 0;
  const int* skip = nullptr;  // optional device flag: non-zero => the launch is a no-op
};

// Epilogues ------------------------------------------------------------------------
struct EpiStore {
  __device__ __forceinline__ double operator()(double v, int64_t, int64_t) const { return v; }
};

// TwoTermPrecond::solve's divide (stk/sylvester.hpp:172-174): wt(i,j) /= lambda_i + theta_j.
struct EpiDivide {
  const double* lam;
  const double* theta;
  __device__ __forceinline__ double operator()(double v, int64_t r, int64_t c) const {
    return v / (lam[r] + theta[c]);
  }
};

// Tile configuration ---------------------------------------------------------------
template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, int MINB_>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int kMinBlocks = MINB_;
  static constexpr int kWarpsM = BM / WM, kWarpsN = BN / WN;
  static constexpr int kThreads = 32 * kWarpsM * kWarpsN;
  // Both tiles are stored k-major, sA[k][perm(m)], sB[k][perm(n)], where perm interleaves
  // rows r and r+8 of every 16-row group (perm(r) = 16*(r/16) + 2*(r%8) + (r/8)%2) so that
  // a thread's two fragment values are one 16-byte shared load.  The pitch (tile + 4
  // doubles) is 8 banks mod 32 per k row: the 128-bit fragment loads are conflict-free.
  static constexpr int kLdsA = BM + 4;
  static constexpr int kLdsB = BN + 4;
  static constexpr int kStageA = BK * kLdsA;
  static constexpr int kStageB = BK * kLdsB;
  static constexpr size_t kSmemBytes = size_t(STAGES) * (kStageA + kStageB) * sizeof(double);
  static constexpr int kMi = WM / 16, kNi = WN / 8;
  static constexpr int kLoadA = BM * BK / kThreads;
  static constexpr int kLoadB = BN * BK / kThreads;
  static_assert(BM * BK % kThreads == 0 && BN * BK % kThreads == 0, "tile/thread mismatch");
  static_assert(BK % 4 == 0 && WM % 16 == 0 && WN % 16 == 0, "mma shape");
};

// 64x64x32 tiles, 4 warps of 32x32, 2 stages, 3 CTAs/SM: the independent CTAs' barrier and
// load phases interleave on each SM, which keeps the DMMA pipe busier than one 256-thread
// 128x128 CTA.  Config sweep on B200 (tools/microbench/gemm_bench.cu,
// profiles/r01_gemm_config_sweep.txt): 32.9 / 32.6 / 26.4 TFLOP/s on the heat left,
// heat batched-right and single 1k^3 (wave preconditioner) shapes vs 28.5 / 28.5 / 12.0
// for 128x128x16.
using GemmTile = GemmCfg<64, 64, 32, 32, 32, 2, 3>;

__host__ __device__ constexpr int perm16(int r) { return (r & ~15) | ((r & 7) << 1) | ((r >> 3) & 1); }

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 8 : 0;  // 0 => zero-fill, nothing read
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// D = A(16x4, row) * B(4x8, col) + C, FP64.  Fragment layout (PTX ISA, mma.m16n8k4 .f64):
// g = lane/4, t = lane%4; a0 = A[g][t], a1 = A[g+8][t]; b0 = B[t][g];
// c0,c1 = C[g][2t, 2t+1], c2,c3 = C[g+8][2t, 2t+1].
__device__ __forceinline__ void dmma_m16n8k4(double (&c)[4], double a0, double a1, double b) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

// One output tile (tm, tn) of batch bt, K-tiles [kt0, kt1), accumulated into acc (zeroed
// here).  Shared by the one-tile-per-CTA kernel and the stream-K kernel.
template <class Cfg>
__device__ __forceinline__ void gemm_tile_accumulate(const GemmProblem& p, int64_t tm, int64_t tn,
                                                     int64_t bt, int64_t kt0, int64_t kt1,
                                                     double* smem,
                                                     double (&acc)[Cfg::kMi][Cfg::kNi][4]) {
  double* sA = smem;                                   // [STAGES][BK][kLdsA]
  double* sB = smem + Cfg::STAGES * Cfg::kStageA;      // [STAGES][BN][kLdsB]
  const int64_t m0 = tm * Cfg::BM, n0 = tn * Cfg::BN;
  const double* A = p.A + bt * p.strideA;
  const double* B = p.B + bt * p.strideB;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % Cfg::kWarpsM, wn = warp / Cfg::kWarpsM;

  // Per-thread load geometry, fixed for the whole K loop: thread tid copies A rows
  // (m = tid % BM, k = tid / BM + i * kRowsA) and B entries (k = tid % BK,
  // n = tid / BK + i * kColsB).  Only one 64-bit product per stage is left in the loop.
  constexpr int kRowsA = Cfg::kThreads / Cfg::BM;
  constexpr int kColsB = Cfg::kThreads / Cfg::BK;
  static_assert(Cfg::kThreads % Cfg::BM == 0 && Cfg::kThreads % Cfg::BK == 0, "load geometry");
  const int am = tid % Cfg::BM, ak = tid / Cfg::BM;
  const int bk = tid % Cfg::BK, bn = tid / Cfg::BK;
  const bool a_row_ok = m0 + am < p.M;
  uint32_t b_col_ok = 0;
#pragma unroll
  for (int i = 0; i < Cfg::kLoadB; ++i)
    if (n0 + bn + i * kColsB < p.N) b_col_ok |= 1u << i;
  const double* a_src = A + (a_row_ok ? m0 + am : 0) + int64_t(ak) * p.lda;
  const double* b_src = B + (b_col_ok & 1u ? (n0 + bn) * p.ldb : 0) + bk;
  const int64_t a_step = int64_t(kRowsA) * p.lda;
  const int64_t b_step = int64_t(kColsB) * p.ldb;
  const int a_dst = ak * Cfg::kLdsA + perm16(am);
  // B entries: n = bn + i * kColsB with bn < kColsB (a power of two): the bits of bn and of
  // i * kColsB are disjoint and perm16 is a bit permutation, so perm16(n) splits into
  // perm16(bn) + perm16(i * kColsB), a compile-time offset per i.
  static_assert((kColsB & (kColsB - 1)) == 0, "kColsB must be a power of two");
  const int b_dst = bk * Cfg::kLdsB + perm16(bn);

  const int64_t kfull = p.K / Cfg::BK;

  auto load_stage = [&](int stage, int64_t kt) {
    const int64_t k0 = kt * Cfg::BK;
    const bool full = kt < kfull;
    double* sa = sA + stage * Cfg::kStageA + a_dst;
    double* sb = sB + stage * Cfg::kStageB + b_dst;
    const double* pa = a_src + k0 * p.lda;
    const double* pb = b_src + k0;
#pragma unroll
    for (int i = 0; i < Cfg::kLoadA; ++i) {
      const bool ok = a_row_ok && (full || k0 + ak + i * kRowsA < p.K);
      cp_async8(sa + i * kRowsA * Cfg::kLdsA, ok ? pa + i * a_step : A, ok);
    }
#pragma unroll
    for (int i = 0; i < Cfg::kLoadB; ++i) {
      const bool ok = ((b_col_ok >> i) & 1u) && (full || k0 + bk < p.K);
      cp_async8(sb + perm16(i * kColsB), ok ? pb + i * b_step : B, ok);
    }
  };

#pragma unroll
  for (int mi = 0; mi < Cfg::kMi; ++mi)
#pragma unroll
    for (int ni = 0; ni < Cfg::kNi; ++ni)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[mi][ni][r] = 0.0;

  const int64_t nk = kt1 - kt0;
#pragma unroll
  for (int s = 0; s < Cfg::STAGES - 1; ++s) {
    if (s < nk) load_stage(s, kt0 + s);
    cp_async_commit();
  }

  // fragments double-buffered across the k4 sub-steps of a stage
  double af[2][Cfg::kMi][2], bf[2][Cfg::kNi];
  auto load_frags = [&](int buf, const double* a_s, const double* b_s, int kk) {
    const double* a_row = a_s + (kk * 4 + t) * Cfg::kLdsA + wm * Cfg::WM + 2 * g;
#pragma unroll
    for (int mi = 0; mi < Cfg::kMi; ++mi) {  // rows g, g+8 of the 16-row group
      const double2 v = *reinterpret_cast<const double2*>(a_row + mi * 16);
      af[buf][mi][0] = v.x;
      af[buf][mi][1] = v.y;
    }
    const double* b_row = b_s + (kk * 4 + t) * Cfg::kLdsB + wn * Cfg::WN + 2 * g;
#pragma unroll
    for (int nj = 0; nj < Cfg::kNi / 2; ++nj) {  // columns g + 16 nj, g + 16 nj + 8
      const double2 v = *reinterpret_cast<const double2*>(b_row + nj * 16);
      bf[buf][2 * nj] = v.x;
      bf[buf][2 * nj + 1] = v.y;
    }
  };

  for (int64_t i = 0; i < nk; ++i) {
    cp_async_wait<Cfg::STAGES - 2>();
    __syncthreads();
    const int stage = static_cast<int>(i % Cfg::STAGES);
    const double* a_s = sA + stage * Cfg::kStageA;
    const double* b_s = sB + stage * Cfg::kStageB;
    load_frags(0, a_s, b_s, 0);
#pragma unroll
    for (int kk = 0; kk < Cfg::BK / 4; ++kk) {
      const int cur = kk & 1;
      if (kk + 1 < Cfg::BK / 4) load_frags(cur ^ 1, a_s, b_s, kk + 1);
#pragma unroll
      for (int mi = 0; mi < Cfg::kMi; ++mi)
#pragma unroll
        for (int ni = 0; ni < Cfg::kNi; ++ni)
          dmma_m16n8k4(acc[mi][ni], af[cur][mi][0], af[cur][mi][1], bf[cur][ni]);
      if (kk == 0) {
        // refill the stage consumed in the previous iteration while the tensor pipe
        // works through the first sub-step's DMMAs
        const int64_t nx = i + Cfg::STAGES - 1;
        if (nx < nk) load_stage(static_cast<int>(nx % Cfg::STAGES), kt0 + nx);
        cp_async_commit();
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // the shared stages may be refilled by the caller's next tile
}

// Epilogue: direct stores (each quad of lanes writes 2 adjacent columns of 8 rows).
template <class Cfg, class Epi>
__device__ __forceinline__ void gemm_tile_store(const GemmProblem& p, int64_t tm, int64_t tn,
                                                int64_t bt, const Epi& epi,
                                                const double (&acc)[Cfg::kMi][Cfg::kNi][4]) {
  double* C = p.C + bt * p.strideC;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % Cfg::kWarpsM, wn = warp / Cfg::kWarpsM;
  const int64_t m0 = tm * Cfg::BM, n0 = tn * Cfg::BN;
#pragma unroll
  for (int mi = 0; mi < Cfg::kMi; ++mi) {
#pragma unroll
    for (int ni = 0; ni < Cfg::kNi; ++ni) {
      const int64_t r0 = m0 + wm * Cfg::WM + mi * 16 + g;
      const int64_t c0 = n0 + wn * Cfg::WN + ni * 8 + 2 * t;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t r = r0 + (q >> 1) * 8;
        const int64_t c = c0 + (q & 1);
        if (r < p.M && c < p.N) C[c * p.ldc + r] = epi(acc[mi][ni][q], r, c);
      }
    }
  }
}

// (the one-tile-per-CTA kernel keeps its own monolithic body: routing it through
// gemm_tile_accumulate / gemm_tile_store measured 6% slower on the heat DMMA transforms)
template <class Cfg, class Epi>
__global__ void __launch_bounds__(Cfg::kThreads, Cfg::kMinBlocks)
    gemm_f64_kernel(const GemmProblem p, const Epi epi) {
  if (p.skip && *p.skip) return;  // device-side early exit (converged Krylov iteration)
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;                                   // [STAGES][BK][kLdsA]
  double* sB = smem + Cfg::STAGES * Cfg::kStageA;      // [STAGES][BN][kLdsB]

  const int64_t tiles_m = (p.M + Cfg::BM - 1) / Cfg::BM;
  const int64_t tiles_n = (p.N + Cfg::BN - 1) / Cfg::BN;
  int64_t bid = blockIdx.x;
  const int64_t tm = bid % tiles_m;
  bid /= tiles_m;
  const int64_t tn = bid % tiles_n;
  const int64_t bt = bid / tiles_n;
  const int64_t m0 = tm * Cfg::BM, n0 = tn * Cfg::BN;

  const double* A = p.A + bt * p.strideA;
  const double* B = p.B + bt * p.strideB;
  double* C = p.C + bt * p.strideC;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % Cfg::kWarpsM, wn = warp / Cfg::kWarpsM;

  // Per-thread load geometry, fixed for the whole K loop: thread tid copies A rows
  // (m = tid % BM, k = tid / BM + i * kRowsA) and B entries (k = tid % BK,
  // n = tid / BK + i * kColsB).  Only one 64-bit product per stage is left in the loop.
  constexpr int kRowsA = Cfg::kThreads / Cfg::BM;
  constexpr int kColsB = Cfg::kThreads / Cfg::BK;
  static_assert(Cfg::kThreads % Cfg::BM == 0 && Cfg::kThreads % Cfg::BK == 0, "load geometry");
  const int am = tid % Cfg::BM, ak = tid / Cfg::BM;
  const int bk = tid % Cfg::BK, bn = tid / Cfg::BK;
  const bool a_row_ok = m0 + am < p.M;
  uint32_t b_col_ok = 0;
#pragma unroll
  for (int i = 0; i < Cfg::kLoadB; ++i)
    if (n0 + bn + i * kColsB < p.N) b_col_ok |= 1u << i;
  const double* a_src = A + (a_row_ok ? m0 + am : 0) + int64_t(ak) * p.lda;
  const double* b_src = B + (b_col_ok & 1u ? (n0 + bn) * p.ldb : 0) + bk;
  const int64_t a_step = int64_t(kRowsA) * p.lda;
  const int64_t b_step = int64_t(kColsB) * p.ldb;
  const int a_dst = ak * Cfg::kLdsA + perm16(am);
  // B entries: n = bn + i * kColsB with bn < kColsB (a power of two): the bits of bn and of
  // i * kColsB are disjoint and perm16 is a bit permutation, so perm16(n) splits into
  // perm16(bn) + perm16(i * kColsB), a compile-time offset per i.
  static_assert((kColsB & (kColsB - 1)) == 0, "kColsB must be a power of two");
  const int b_dst = bk * Cfg::kLdsB + perm16(bn);

  const int64_t ktiles = (p.K + Cfg::BK - 1) / Cfg::BK;
  const int64_t kfull = p.K / Cfg::BK;

  auto load_stage = [&](int stage, int64_t kt) {
    const int64_t k0 = kt * Cfg::BK;
    const bool full = kt < kfull;
    double* sa = sA + stage * Cfg::kStageA + a_dst;
    double* sb = sB + stage * Cfg::kStageB + b_dst;
    const double* pa = a_src + k0 * p.lda;
    const double* pb = b_src + k0;
#pragma unroll
    for (int i = 0; i < Cfg::kLoadA; ++i) {
      const bool ok = a_row_ok && (full || k0 + ak + i * kRowsA < p.K);
      cp_async8(sa + i * kRowsA * Cfg::kLdsA, ok ? pa + i * a_step : A, ok);
    }
#pragma unroll
    for (int i = 0; i < Cfg::kLoadB; ++i) {
      const bool ok = ((b_col_ok >> i) & 1u) && (full || k0 + bk < p.K);
      cp_async8(sb + perm16(i * kColsB), ok ? pb + i * b_step : B, ok);
    }
  };

  double acc[Cfg::kMi][Cfg::kNi][4];
#pragma unroll
  for (int mi = 0; mi < Cfg::kMi; ++mi)
#pragma unroll
    for (int ni = 0; ni < Cfg::kNi; ++ni)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[mi][ni][r] = 0.0;

#pragma unroll
  for (int s = 0; s < Cfg::STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_async_commit();
  }

  // fragments double-buffered across the k4 sub-steps of a stage
  double af[2][Cfg::kMi][2], bf[2][Cfg::kNi];
  auto load_frags = [&](int buf, const double* a_s, const double* b_s, int kk) {
    const double* a_row = a_s + (kk * 4 + t) * Cfg::kLdsA + wm * Cfg::WM + 2 * g;
#pragma unroll
    for (int mi = 0; mi < Cfg::kMi; ++mi) {  // rows g, g+8 of the 16-row group
      const double2 v = *reinterpret_cast<const double2*>(a_row + mi * 16);
      af[buf][mi][0] = v.x;
      af[buf][mi][1] = v.y;
    }
    const double* b_row = b_s + (kk * 4 + t) * Cfg::kLdsB + wn * Cfg::WN + 2 * g;
#pragma unroll
    for (int nj = 0; nj < Cfg::kNi / 2; ++nj) {  // columns g + 16 nj, g + 16 nj + 8
      const double2 v = *reinterpret_cast<const double2*>(b_row + nj * 16);
      bf[buf][2 * nj] = v.x;
      bf[buf][2 * nj + 1] = v.y;
    }
  };

  for (int64_t kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<Cfg::STAGES - 2>();
    __syncthreads();
    const int stage = static_cast<int>(kt % Cfg::STAGES);
    const double* a_s = sA + stage * Cfg::kStageA;
    const double* b_s = sB + stage * Cfg::kStageB;
    load_frags(0, a_s, b_s, 0);
#pragma unroll
    for (int kk = 0; kk < Cfg::BK / 4; ++kk) {
      const int cur = kk & 1;
      if (kk + 1 < Cfg::BK / 4) load_frags(cur ^ 1, a_s, b_s, kk + 1);
#pragma unroll
      for (int mi = 0; mi < Cfg::kMi; ++mi)
#pragma unroll
        for (int ni = 0; ni < Cfg::kNi; ++ni)
          dmma_m16n8k4(acc[mi][ni], af[cur][mi][0], af[cur][mi][1], bf[cur][ni]);
      if (kk == 0) {
        // refill the stage consumed in the previous iteration while the tensor pipe
        // works through the first sub-step's DMMAs
        const int64_t nk = kt + Cfg::STAGES - 1;
        if (nk < ktiles) load_stage(static_cast<int>(nk % Cfg::STAGES), nk);
        cp_async_commit();
      }
    }
  }
  cp_async_wait<0>();

  // Epilogue: direct stores (each quad of lanes writes 2 adjacent columns of 8 rows).
#pragma unroll
  for (int mi = 0; mi < Cfg::kMi; ++mi) {
#pragma unroll
    for (int ni = 0; ni < Cfg::kNi; ++ni) {
      const int64_t r0 = m0 + wm * Cfg::WM + mi * 16 + g;
      const int64_t c0 = n0 + wn * Cfg::WN + ni * 8 + 2 * t;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t r = r0 + (q >> 1) * 8;
        const int64_t c = c0 + (q & 1);
        if (r < p.M && c < p.N) C[c * p.ldc + r] = epi(acc[mi][ni][q], r, c);
      }
    }
  }
}

// ---------------------------------------------------------------------------- stream-K --
// Persistent stream-K schedule for single GEMMs whose tile count leaves CTA slots idle (the
// 1023 x 1023 x 1025 wave preconditioner products: 272 tiles of 64 x 64 for 444 slots).  The
// (tile, K-tile) iteration space is cut into G equal contiguous ranges, one per resident CTA
// (G = the occupancy-limited slot count, so every CTA is resident and the flag waits below
// cannot deadlock).  A tile split across CTAs is finished by the CTA holding its first
// K-tiles, which reaches them at the END of its range -- the later segments' CTAs met theirs at
// the start of their ranges, so the finisher rarely waits (finishing on the last segment
// instead would make that CTA idle through its predecessor's whole range).  The other segments
// store their accumulators to a workspace slot and publish a flag (the launch's epoch); the
// finisher adds the slots in segment order (deterministic) and applies the epilogue.
struct StreamKWork {
  double* partials = nullptr;   // tiles * kMaxSeg * BM * BN doubles
  unsigned* flags = nullptr;    // tiles * kMaxSeg
  int64_t tiles_cap = 0;
  unsigned epoch = 0;
  static constexpr int kMaxSeg = 4;
};

template <class Cfg, class Epi>
__global__ void __launch_bounds__(Cfg::kThreads, Cfg::kMinBlocks)
    gemm_f64_streamk_kernel(const GemmProblem p, const Epi epi, double* __restrict__ partials,
                            unsigned* __restrict__ flags, unsigned epoch) {
  if (p.skip && *p.skip) return;
  extern __shared__ __align__(16) double smem[];
  constexpr int kFrag = Cfg::kMi * Cfg::kNi * 4;
  const int64_t tiles_m = (p.M + Cfg::BM - 1) / Cfg::BM;
  const int64_t tiles_n = (p.N + Cfg::BN - 1) / Cfg::BN;
  const int64_t ktiles = (p.K + Cfg::BK - 1) / Cfg::BK;
  const int64_t W = tiles_m * tiles_n * ktiles;
  const int64_t G = gridDim.x, c = blockIdx.x;
  auto start = [&](int64_t cc) { return cc * W / G; };
  const int64_t u_end = start(c + 1);
  double acc[Cfg::kMi][Cfg::kNi][4];
  for (int64_t u = start(c); u < u_end;) {
    const int64_t tile = u / ktiles, kt0 = u - tile * ktiles;
    const int64_t kt1 = (tile + 1) * ktiles < u_end ? ktiles : u_end - tile * ktiles;
    const int64_t tm = tile % tiles_m, tn = tile / tiles_m;
    gemm_tile_accumulate<Cfg>(p, tm, tn, 0, kt0, kt1, smem, acc);
    // segments of the tile: CTAs c0 .. c1 (owners of its first and last K-tile); this CTA is
    // segment c - c0, the finisher is segment 0 (kt0 == 0)
    auto owner = [&](int64_t uu) {
      int64_t cc = uu * G / W;
      while (start(cc + 1) <= uu) ++cc;
      while (start(cc) > uu) --cc;
      return cc;
    };
    const int64_t c0 = owner(tile * ktiles), c1 = owner(tile * ktiles + ktiles - 1);
    const int seg = static_cast<int>(c - c0), nseg = static_cast<int>(c1 - c0 + 1);
    double* slot_base = partials + (tile * StreamKWork::kMaxSeg) * int64_t(kFrag) * Cfg::kThreads;
    unsigned* flag_base = flags + tile * StreamKWork::kMaxSeg;
    if (kt0 == 0 && kt1 == ktiles) {
      gemm_tile_store<Cfg>(p, tm, tn, 0, epi, acc);
    } else if (kt0 > 0) {  // not the finisher: publish the partial sums
      double* slot = slot_base + int64_t(seg) * kFrag * Cfg::kThreads;
      int f = 0;
#pragma unroll
      for (int mi = 0; mi < Cfg::kMi; ++mi)
#pragma unroll
        for (int ni = 0; ni < Cfg::kNi; ++ni)
#pragma unroll
          for (int r = 0; r < 4; ++r, ++f) __stcg(slot + f * Cfg::kThreads + threadIdx.x, acc[mi][ni][r]);
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(flag_base + seg), "r"(epoch)
                     : "memory");
      }
    } else {  // finisher (segment 0): add the later segments in order, then the epilogue
      if (threadIdx.x >= 1 && threadIdx.x < nseg) {
        unsigned v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n"
                       : "=r"(v)
                       : "l"(flag_base + threadIdx.x)
                       : "memory");
        } while (v != epoch);
      }
      __syncthreads();
      double tot[Cfg::kMi][Cfg::kNi][4];
#pragma unroll
      for (int mi = 0; mi < Cfg::kMi; ++mi)
#pragma unroll
        for (int ni = 0; ni < Cfg::kNi; ++ni)
#pragma unroll
          for (int r = 0; r < 4; ++r) tot[mi][ni][r] = 0.0;
      for (int sg = 1; sg < nseg; ++sg) {
        const double* slot = slot_base + int64_t(sg) * kFrag * Cfg::kThreads;
        int f = 0;
#pragma unroll
        for (int mi = 0; mi < Cfg::kMi; ++mi)
#pragma unroll
          for (int ni = 0; ni < Cfg::kNi; ++ni)
#pragma unroll
            for (int r = 0; r < 4; ++r, ++f)
              tot[mi][ni][r] += __ldcg(slot + f * Cfg::kThreads + threadIdx.x);
      }
#pragma unroll
      for (int mi = 0; mi < Cfg::kMi; ++mi)
#pragma unroll
        for (int ni = 0; ni < Cfg::kNi; ++ni)
#pragma unroll
          for (int r = 0; r < 4; ++r) tot[mi][ni][r] += acc[mi][ni][r];
      gemm_tile_store<Cfg>(p, tm, tn, 0, epi, tot);
    }
    u = tile * ktiles + kt1;
  }
}

template <class Cfg, class Epi>
void launch_gemm_cfg(const GemmProblem& p, const Epi& epi, cudaStream_t stream) {
  static const bool configured = [] {  // thread-safe one-time opt-in to >48 KB smem
    STKG_CUDA_CHECK(cudaFuncSetAttribute(gemm_f64_kernel<Cfg, Epi>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(Cfg::kSmemBytes)));
    return true;
  }();
  (void)configured;
  const int64_t blocks = ceil_div(p.M, Cfg::BM) * ceil_div(p.N, Cfg::BN) * p.batch;
  STKG_REQUIRE(blocks < (int64_t(1) << 31), STKG_ARGUMENT, "gemm: grid too large");
  if (blocks == 0) return;
  gemm_f64_kernel<Cfg, Epi><<<static_cast<unsigned>(blocks), Cfg::kThreads, Cfg::kSmemBytes,
                              stream>>>(p, epi);
  STKG_CUDA_CHECK(cudaGetLastError());
}

template <class Epi>
void launch_gemm(const GemmProblem& p, const Epi& epi, cudaStream_t stream) {
  launch_gemm_cfg<GemmTile>(p, epi, stream);
}

// Stream-K launch for a single (batch 1) GEMM when its tiles would leave CTA slots idle
// (opt-in, STKG_STREAMK=1: measured slower than one tile per CTA at the 1k^3 wave shape,
// 0.296 vs 0.262 ms per modal preconditioner solve -- DESIGN.md K2); falls back to the
// one-tile-per-CTA kernel otherwise.  ws is the caller's workspace (grown here; the
// caller's stream orders its reuse).
template <class Epi>
void launch_gemm_streamk(const GemmProblem& p, const Epi& epi, cudaStream_t stream,
                         StreamKWork& ws) {
  using Cfg = GemmTile;
  static const bool enabled = [] {
    const char* e = std::getenv("STKG_STREAMK");
    return e && e[0] == '1';
  }();
  static const int per_sm = [] {
    STKG_CUDA_CHECK(cudaFuncSetAttribute(gemm_f64_streamk_kernel<Cfg, Epi>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(Cfg::kSmemBytes)));
    int b = 0;
    STKG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &b, gemm_f64_streamk_kernel<Cfg, Epi>, Cfg::kThreads, Cfg::kSmemBytes));
    return std::max(b, 1);
  }();
  const int64_t tiles = ceil_div(p.M, Cfg::BM) * ceil_div(p.N, Cfg::BN);
  const int64_t ktiles = ceil_div(p.K, Cfg::BK);
  const int64_t slots = int64_t(num_sms()) * per_sm;
  if (!enabled || p.batch != 1 || tiles >= slots || tiles == 0 ||
      ktiles * tiles < slots * 2) {
    launch_gemm(p, epi, stream);
    return;
  }
  constexpr int kFrag = Cfg::kMi * Cfg::kNi * 4;
  if (ws.tiles_cap < tiles) {
    STKG_CUDA_CHECK(cudaStreamSynchronize(stream));
    if (ws.partials) STKG_CUDA_CHECK(cudaFree(ws.partials));
    if (ws.flags) STKG_CUDA_CHECK(cudaFree(ws.flags));
    STKG_CUDA_CHECK(cudaMalloc(&ws.partials, sizeof(double) * tiles * StreamKWork::kMaxSeg *
                                                 kFrag * Cfg::kThreads));
    STKG_CUDA_CHECK(cudaMalloc(&ws.flags, sizeof(unsigned) * tiles * StreamKWork::kMaxSeg));
    STKG_CUDA_CHECK(cudaMemsetAsync(ws.flags, 0, sizeof(unsigned) * tiles * StreamKWork::kMaxSeg,
                                    stream));
    ws.tiles_cap = tiles;
  }
  // every split tile has at most kMaxSeg segments: each CTA's range covers >= 2 K-tiles' worth
  STKG_REQUIRE(ktiles * tiles / slots >= (ktiles + StreamKWork::kMaxSeg - 2) / (StreamKWork::kMaxSeg - 1),
               STKG_ARGUMENT, "stream-K: too many segments per tile");
  ws.epoch = ws.epoch + 1 == 0 ? 1 : ws.epoch + 1;
  gemm_f64_streamk_kernel<Cfg, Epi><<<static_cast<unsigned>(slots), Cfg::kThreads,
                                      Cfg::kSmemBytes, stream>>>(p, epi, ws.partials, ws.flags,
                                                                 ws.epoch);
  STKG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace stkg
