// Half-length fast sine transform (DST-I) for the uniform-P1 eigenbasis.
//
// dst.cuh transforms two real vectors with one complex FFT of length 2N (N = n + 1).  The
// kernels here need a complex FFT of length N for the same two vectors -- half the flops
// and half the shared-memory traffic -- by the classical odd-symmetry reduction of DST-I
// to a real DFT of length N:
//
//     y_0 = 0,  y_j = sin(pi j / N) (x_j + x_{N-j}) + (x_j - x_{N-j}) / 2   (j = 1..N-1)
//     Y_k = sum_j y_j exp(-2 pi i j k / N) = A_k - i B_k
//     DST(x)_{2k}   = B_k                          (k = 1..N/2-1)
//     DST(x)_{2k+1} = DST(x)_{2k-1} + A_k,  DST(x)_1 = A_0 / 2   (k = 0..N/2-1)
//
// (the x_{N-j} terms cancel in B and double in A; sin(pi j/N) cos(2 pi j k/N) splits into
// the two neighbouring odd sines).  Two real vectors a, b share one complex FFT
// z = y(a) + i y(b): Y(a)_k = (Z_k + conj Z_{N-k}) / 2, Y(b)_k = (Z_k - conj Z_{N-k}) / 2i.
// The odd outputs are a prefix sum over k: serial within a thread (consecutive k), one
// warp-shuffle block scan across threads.  Its rounding grows like sqrt(N) eps.
//
// FFT: Stockham auto-sort in shared memory with every thread holding V = 16 complex
// values; a stage of radix R <= V runs V/R butterflies per thread.  All stages read the
// thread's values from positions t + T p (T = N/V threads per FFT, p < V), so one read
// pattern serves every stage; pidx() padding spreads the stride-T accesses over banks.
// Twiddles come from the 2N-th-root table the plan already holds (stride 2), and
// sin(pi m / N) = -Im of its m-th entry.
//
// Used by 2D/3D plans for N in [16, 1024] (heat.cu::dst_pass).  FFTs with T <= 32 threads
// are aligned lane segments (several per warp, warp-level barriers and segmented shuffles);
// T = 64 (N = 1024) spans two warps.  N = 2048 and 1D plans keep the dst.cuh kernels.
#pragma once

#ifndef STKG_HALF_V
#define STKG_HALF_V 16
#endif

#include <cuda.h>  // CUtensorMap (the TMA descriptor type; the encoder is fetched at run time)

#include "dst.cuh"

namespace stkg {

template <int R>
__device__ __forceinline__ void dft_small(double2 (&u)[R]);
template <>
__device__ __forceinline__ void dft_small<2>(double2 (&u)[2]) { dft_radix<2>(u); }
template <>
__device__ __forceinline__ void dft_small<4>(double2 (&u)[4]) { dft_radix<4>(u); }
template <>
__device__ __forceinline__ void dft_small<8>(double2 (&u)[8]) { dft8(u); }
template <>
__device__ __forceinline__ void dft_small<16>(double2 (&u)[16]) {
  // 16 = 2 x 8 by decimation in frequency: a_r = u_r + u_{r+8}, b_r = (u_r - u_{r+8}) w16^r,
  // two DFT-8, outputs even <- a, odd <- b.
  constexpr double c1 = 0.92387953251128675613;  // cos(pi/8)
  constexpr double s1 = 0.38268343236508977173;  // sin(pi/8)
  constexpr double r2 = 0.70710678118654752440;
  double2 a[8], b[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    a[r] = cadd(u[r], u[r + 8]);
    b[r] = csub(u[r], u[r + 8]);
  }
  b[1] = cmul(b[1], make_double2(c1, -s1));
  b[2] = make_double2((b[2].x + b[2].y) * r2, (b[2].y - b[2].x) * r2);
  b[3] = cmul(b[3], make_double2(s1, -c1));
  b[4] = mul_neg_i(b[4]);
  b[5] = cmul(b[5], make_double2(-s1, -c1));
  b[6] = make_double2((b[6].y - b[6].x) * r2, -(b[6].x + b[6].y) * r2);
  b[7] = cmul(b[7], make_double2(-c1, -s1));
  dft8(a);
  dft8(b);
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    u[2 * p] = a[p];
    u[2 * p + 1] = b[p];
  }
}

// L2 prefetch of a later work item (STKG_DST_PREFETCH items ahead, 0 = off) while the
// current one computes, with no registers held: its global loads then hit L2 instead of
// waiting on DRAM.  Measured on the contiguous kernel: 271.5 / 279.6 -> 262.1 / 268.3 us
// per 64-slice cfg3 pass (fwd / inv); on the strided kernel (cp.async staging) neutral.
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}
#ifndef STKG_DST_PREFETCH
#define STKG_DST_PREFETCH 1
#endif

// Barrier over the threads of one FFT: a warp barrier when the FFT fits in one warp (its
// shared region is private to the warp's FFTs), else a CTA barrier.
// bar > 0: the FFT's own named barrier (bar.sync bar, T) so that several FFTs of one CTA
// do not wait for each other inside their stages; bar == 0: the CTA barrier.
template <int T>
__device__ __forceinline__ void fft_sync(int bar = 0) {
  if constexpr (T <= 32) {  // FFTs are aligned lane segments: the warp runs them in lockstep
    __syncwarp();
  } else {
    if (bar > 0) {
      asm volatile("bar.sync %0, %1;\n" ::"r"(bar), "n"(T) : "memory");
    } else {
      __syncthreads();
    }
  }
}

// Shared-memory index of the half-length FFT buffer: an XOR swizzle of the low three bits
// (a permutation inside aligned groups of 8 complex = 128 bytes).  Checked offline against
// every access pattern of the kernels (first-stage writes of 16 consecutive values per
// thread, the t + T p reads, the later stage writes and the post-processing's k and N - k
// reads): conflict-free for 128-bit accesses except 1/8 of the N - k reads (2-way).
__host__ __device__ constexpr int hpidx(int i) { return i ^ (((i >> 3) ^ (i >> 6)) & 7); }
// Buffer length (complex): N for the FFT, and 2 opad(N) doubles for the output staging.
template <int N>
constexpr int hpadded_len() { return N + N / (STKG_HALF_V < 16 ? STKG_HALF_V : 16); }

// One Stockham stage (radix R; NS = product of the earlier radices) of a length-N FFT
// whose T = N/V threads hold x[p] = value at position t + T p.  Computes in registers,
// writes the stage output to buf, and re-reads the thread's values for the next stage.
// LIN: this stage's output goes to buf in linear order (no swizzle) -- used for the stage
// that feeds the fused last stage (half_fft_post), whose mirrored reads (N - k runs, not
// 8-aligned) would straddle two swizzle groups and conflict 2-way; with NS >= 8 this
// stage's writes (8 consecutive j per quarter-warp phase) are conflict-free in linear order.
template <int N, int V, int R, int NS, bool LIN = false>
__device__ __forceinline__ void half_stage(double2 (&x)[V], double2* buf,
                                           const double2* __restrict__ tw2, int t, int bar) {
  constexpr int T = N / V;
  constexpr int B = V / R;                   // butterflies per thread
  constexpr int kStep = (2 * N) / (NS * R);  // tw2 index of exp(-2 pi i / (NS R))
#pragma unroll
  for (int i = 0; i < B; ++i) {
    const int j = t + T * i;
    const int k = j % NS;
    double2 u[R];
#pragma unroll
    for (int q = 0; q < R; ++q) u[q] = x[i + q * B];
    if constexpr (NS > 1) {
      if (k > 0) {
        const double2 w = __ldg(tw2 + k * kStep);
        double2 wr = w;
#pragma unroll
        for (int q = 1; q < R; ++q) {
          if (q > 1) wr = cmul(wr, w);
          u[q] = cmul(u[q], wr);
        }
      }
    }
    dft_small<R>(u);
#pragma unroll
    for (int q = 0; q < R; ++q) x[i + q * B] = u[q];
  }
  fft_sync<T>(bar);  // every thread has consumed the previous contents of buf
#pragma unroll
  for (int i = 0; i < B; ++i) {
    const int j = t + T * i;
    const int base = (j / NS) * NS * R + j % NS;
#pragma unroll
    for (int q = 0; q < R; ++q) buf[LIN ? base + q * NS : hpidx(base + q * NS)] = x[i + q * B];
  }
  fft_sync<T>(bar);
  if constexpr (NS * R < N && !LIN) {  // the last stage's output is consumed from buf directly
#pragma unroll
    for (int p = 0; p < V; ++p) x[p] = buf[hpidx(t + T * p)];
  }
}

// All stages: radix V while V divides the remaining length, then the remainder radix.
// Stops before the stage whose NS reaches STOP (STOP = N: run them all).
template <int N, int V, int NS, int STOP = N, bool LL = false>
__device__ __forceinline__ void half_fft_stages(double2 (&x)[V], double2* buf,
                                                const double2* __restrict__ tw2, int t, int bar) {
  if constexpr (NS < STOP) {
    constexpr int rem = N / NS;
    constexpr int R = rem >= V ? V : rem;
    constexpr bool LIN = LL && STOP < N && NS * R == STOP && NS >= 8;
    half_stage<N, V, R, NS, LIN>(x, buf, tw2, t, bar);
    half_fft_stages<N, V, NS * R, STOP, LL>(x, buf, tw2, t, bar);
  }
}

// NS of the stage that runs just before the stage with NS = stop.
template <int N, int V>
constexpr int stage_before(int stop) {
  int ns = 1;
  for (;;) {
    const int rem = N / ns, r = rem >= V ? V : rem;
    if (ns * r >= stop) return ns;
    ns *= r;
  }
}

// NS of the last Stockham stage of the length-N plan.
template <int N, int V, int NS = 1>
constexpr int last_stage_ns() {
  if constexpr (N / NS <= V) {
    return NS;
  } else {
    return last_stage_ns<N, V, NS * V>();
  }
}

// Output staging index: one pad double per V (conflict-free for the post-processing
// writes, in which thread t writes V consecutive outputs).
template <int V>
__device__ __forceinline__ int opad(int e) { return e + e / V; }

// Inclusive prefix sum of (a, b) over the T threads of one FFT.  T <= 32: the FFT is an
// aligned segment of T lanes (segmented shuffles); T > 32: whole warps, cross-warp totals
// through red (2 T/32 doubles for this FFT).
template <int T>
__device__ __forceinline__ void fft_scan2(double& a, double& b, double* red, int t, int bar) {
  constexpr int W = T < 32 ? T : 32;
  const int lane = t & (W - 1);
#pragma unroll
  for (int o = 1; o < W; o <<= 1) {
    const double ta = __shfl_up_sync(0xffffffffu, a, o, W);
    const double tb = __shfl_up_sync(0xffffffffu, b, o, W);
    if (lane >= o) {
      a += ta;
      b += tb;
    }
  }
  if constexpr (T > 32) {
    const int warp = t >> 5;
    if (lane == 31) {
      red[2 * warp] = a;
      red[2 * warp + 1] = b;
    }
    fft_sync<T>(bar);
    double oa = 0.0, ob = 0.0;
    for (int w = 0; w < warp; ++w) {
      oa += red[2 * w];
      ob += red[2 * w + 1];
    }
    a += oa;
    b += ob;
  }
}

// Pre-processing of one FFT input position m (value pair x_m, x_{N-m} of both vectors).
__device__ __forceinline__ double2 half_pre(double s, double xa, double xam, double xb,
                                            double xbm) {
  return make_double2(fma(s, xa + xam, 0.5 * (xa - xam)), fma(s, xb + xbm, 0.5 * (xb - xbm)));
}

// Output staging of the n transformed values of both vectors of a pair.
// OutSplit: two arrays of doubles (one per vector) at opad(e), read back per vector by the
// contiguous-axis stores.  OutPair: one array of double2 (a_e, b_e) at idx(e), read back
// as 16-byte rows by the strided 16-byte kernel.
template <int V>
struct OutSplit {
  double* oa;
  double* ob;
  __device__ __forceinline__ void put(int e, double a, double b) const {
    oa[opad<V>(e)] = a;
    ob[opad<V>(e)] = b;
  }
  __device__ __forceinline__ void get(int e, double& a, double& b) const {
    a = oa[opad<V>(e)];
    b = ob[opad<V>(e)];
  }
};
// OFF: the odd half starts at N/2 + OFF (OFF = 4 puts the odd outputs of a k in the other
// half of the bank groups, for readers of 8 consecutive outputs -- heat_fused.cuh).
template <int N, int OFF = 0>
struct OutPair {
  double2* o;
#if STKG_OUTPAIR_LINEAR
  __device__ __forceinline__ static int idx(int e) { return e + (e >> 4); }
#else
  // Even outputs e = 2k at p(k), odd outputs e = 2k - 1 at N/2 + p(k), p(k) = k XOR-swizzled
  // by k / 8 within groups of 64: the post-processing's writes of 8 consecutive k, the
  // scan's reads of k = 8t + i over 8 consecutive t and the tile copy's (even, odd) pairs
  // fall in distinct 16-byte bank groups (the previous e + e/16 layout made every stride-2
  // post-processing write phase 2-way conflicted).
  __device__ __forceinline__ static int idx(int e) {
    const int k = (e + 1) >> 1;
    return (e & 1) * (N / 2 + OFF) + (k ^ ((k >> 3) & 7));
  }
#endif
  __device__ __forceinline__ void put(int e, double a, double b) const { o[idx(e)] = make_double2(a, b); }
  __device__ __forceinline__ void get(int e, double& a, double& b) const {
    const double2 v = o[idx(e)];
    a = v.x;
    b = v.y;
  }
};

// Post-processing of the outputs k < N/2 (a thread owns a set of k and, for each, both
// Z_k and Z_{N-k}): B_k -> X_{2k} at index 2k - 1; A_k parked at index 2k.  Then the
// prefix scan over k: thread t re-reads the A of k = t H .. t H + H - 1 (consecutive),
// scans serially and across threads, and writes X_{2k+1} back to index 2k.
template <int N, int V, class Out>
__device__ __forceinline__ void half_scan_odd(int t, double* red, const Out& out, int bar) {
  constexpr int T = N / V, H = V / 2;
  double Aa[H], Ab[H];
  double sa = 0.0, sb = 0.0;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const int k = t * H + i;
    double a, b;
    out.get(2 * k, a, b);
    sa += a;
    sb += b;
    Aa[i] = sa;
    Ab[i] = sb;
  }
  double ea = sa, eb = sb;
  fft_scan2<T>(ea, eb, red, t, bar);
  ea -= sa;
  eb -= sb;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const int k = t * H + i;
    out.put(2 * k, Aa[i] + ea, Ab[i] + eb);
  }
}

// FFT (x holds the pre-processed inputs), post-processing and prefix scan; writes the
// n outputs of both vectors through out (OutSplit / OutPair).  buf may overlap out.
//
// When the last Stockham stage gives every thread B >= 2 butterflies, it is fused with the
// post-processing: thread t takes the mirrored butterflies j and NS - j (thread 0 the
// multiples of T), so Z_k and Z_{N-k} meet in its registers and the last stage's output
// never goes to shared memory.
// LL: the stage feeding the fused last stage writes linearly (half_stage's LIN); measured
// 1% faster for the contiguous kernel, slower for the strided one (28 bytes of spills).
template <int N, int V, bool LL = false, class Out>
__device__ __forceinline__ void half_fft_post(double2 (&x)[V], double2* buf,
                                             const double2* __restrict__ tw2, int t, double hs,
                                             double* red, const Out& out, int bar = 0) {
  constexpr int T = N / V, H = V / 2;
  constexpr int NSL = last_stage_ns<N, V>();
  constexpr int RL = N / NSL;   // radix of the last stage
  constexpr int BL = NSL / T;   // its butterflies per thread
  if constexpr (BL >= 2 && NSL > 1) {
    // the stage-(L-1) output is left in buf, linear when that stage has NS >= 8
    constexpr bool LINL = LL && stage_before<N, V>(NSL) >= 8;
    half_fft_stages<N, V, 1, NSL, LL>(x, buf, tw2, t, bar);
    // butterflies of this thread: jj[0..BL/2) and their mirrors jj[BL/2 + i] = NSL - jj[i]
    int jj[BL];
#pragma unroll
    for (int i = 0; i < BL / 2; ++i) {
      jj[i] = t == 0 ? T * i : t + T * i;
      jj[BL / 2 + i] = t == 0 ? T * (BL / 2 + i) : NSL - (t + T * i);
    }
    double2 z[BL][RL];
#pragma unroll
    for (int b = 0; b < BL; ++b) {
      const int j = jj[b];
#pragma unroll
      for (int q = 0; q < RL; ++q) z[b][q] = buf[LINL ? j + NSL * q : hpidx(j + NSL * q)];
      if (j > 0) {
        const double2 w = __ldg(tw2 + 2 * j);  // exp(-2 pi i j / N)
        double2 wr = w;
#pragma unroll
        for (int q = 1; q < RL; ++q) {
          if (q > 1) wr = cmul(wr, w);
          z[b][q] = cmul(z[b][q], wr);
        }
      }
      dft_small<RL>(z[b]);  // z[b][q] = Z_{j + NSL q}
    }
    fft_sync<T>(bar);  // every thread has read buf: the output staging may overwrite it
#pragma unroll
    for (int b = 0; b < BL; ++b) {
      const int j = jj[b];
#pragma unroll
      for (int q = 0; q < RL / 2; ++q) {  // k = j + NSL q < N/2
        const int k = j + NSL * q;
        double2 zm;
        if (t == 0) {
          // thread 0 holds the multiples of T: j = T i pairs with NSL - j = T (BL - i)
          // (b < BL/2: i = b; b >= BL/2: i = b); j = 0 and j = NSL/2 pair with themselves
          const int bi = (j == 0) ? b : (BL - b) % BL;
          const int qm = (j == 0) ? (RL - q) % RL : RL - 1 - q;
          zm = z[bi][qm];
        } else {
          const int bm = b < BL / 2 ? b + BL / 2 : b - BL / 2;
          zm = z[bm][RL - 1 - q];
        }
        const double2 zk = z[b][q];
        double Aa = hs * (zk.x + zm.x), Ab = hs * (zk.y + zm.y);
        if (k == 0) {
          Aa *= 0.5;
          Ab *= 0.5;
        } else {
          out.put(2 * k - 1, hs * (zm.y - zk.y), hs * (zk.x - zm.x));
        }
        out.put(2 * k, Aa, Ab);
      }
    }
    fft_sync<T>(bar);
    half_scan_odd<N, V>(t, red, out, bar);
  } else {
    half_fft_stages<N, V, 1>(x, buf, tw2, t, bar);
    // thread t owns k = t H + i (i < H) of the half spectrum k < N/2
    double Aa[H], Ab[H], Ba[H], Bb[H];
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const int k = t * H + i;
      const double2 zk = buf[hpidx(k)];
      const double2 zm = buf[hpidx(k == 0 ? 0 : N - k)];
      Aa[i] = hs * (zk.x + zm.x);
      Ab[i] = hs * (zk.y + zm.y);
      Ba[i] = hs * (zm.y - zk.y);
      Bb[i] = hs * (zk.x - zm.x);
    }
    if (t == 0) {
      Aa[0] *= 0.5;
      Ab[0] *= 0.5;
    }
    double sa = 0.0, sb = 0.0;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      sa += Aa[i];
      sb += Ab[i];
      Aa[i] = sa;
      Ab[i] = sb;
    }
    double ea = sa, eb = sb;
    fft_scan2<T>(ea, eb, red, t, bar);
    ea -= sa;  // exclusive offsets
    eb -= sb;
    fft_sync<T>(bar);  // all reads of Z are done: buf may be overwritten by the outputs
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const int k = t * H + i;
      if (k > 0) out.put(2 * k - 1, Ba[i], Bb[i]);  // X_{2k} -> index 2k - 1
      out.put(2 * k, Aa[i] + ea, Ab[i] + eb);       // X_{2k+1} -> index 2k
    }
  }
}

// Values per thread: 16 (radix-16 stages, then the remainder radix).  A radix-32 variant
// for N = 1024 (two stages, one warp per FFT) measured 9% slower on cfg3 (27.8 vs 25.5 ms:
// 168 registers, 12 warps/SM) and V = 8 15% slower; see DESIGN.md's tuning log.
template <int N>
constexpr int half_v() { return STKG_HALF_V; }

// Contiguous-axis configuration: F FFTs (vector pairs) per CTA so that a CTA has at least
// 64 threads; each FFT owns T = N/V threads (an aligned lane segment when T <= 32).
template <int N>
struct HalfCfg {
  static constexpr int V = half_v<N>();
  static constexpr int T = N / V;             // threads per FFT
  static constexpr int F = T >= 64 ? 1 : 64 / T;  // FFTs per CTA
  static constexpr int kThreads = F * T;
  // complex per FFT buffer.  With T in [2, 8] a half-warp holds 16/T FFTs, whose 8-byte
  // output-staging accesses run in the same phase: the buffers are skewed to kBuf = T/2
  // (mod 8) complex so those FFTs start T 8-byte banks apart (unskewed, every buffer began
  // at the same bank and the puts / scan accesses were 2-way conflicted: 29% excess
  // wavefronts at N = 128, profiles/r02 notes in DESIGN.md K2b).
  static constexpr int kBuf0 = hpadded_len<N>();
  static constexpr int kBuf = (T >= 2 && T <= 8) ? kBuf0 + ((T / 2 - kBuf0 % 8) + 8) % 8 : kBuf0;
  static constexpr size_t kSmem = size_t(F) * kBuf * sizeof(double2);
#ifdef STKG_HALF_MINB
  static constexpr int kMinBlocks = STKG_HALF_MINB;
#else
  static constexpr int kMinBlocks = 65536 / (kThreads * 128) < 8 ? 65536 / (kThreads * 128) : 8;
#endif
  static_assert(T <= 32 || T % 32 == 0, "FFTs are lane segments or whole warps");
};

// Contiguous axis (vector g of length n = N - 1 at src + g ld_src, written to dst + g ld_dst;
// ld = n: back to back): a CTA step transforms F consecutive vector pairs (persistent grid).
// ld_dst > n (the padded internal layout of heat.cu's device solve) also writes zeros into
// the ld_dst - n pad entries, so that the padded lanes stay finite through later passes.
// dst may alias src when ld_src == ld_dst (an item is read completely before it is written).
// ticket != nullptr: items are handed out dynamically (atomicAdd on *ticket, which must be 0
// at launch) instead of by grid stride -- used when the kernel runs beside the fused axis-0
// pass on the SMs that pass leaves idle (heat.cu run_chunk_padded_overlap), where a static
// split would leave the items of not-yet-resident CTAs waiting.
template <int N, bool DYN = false>
__global__ void __launch_bounds__(HalfCfg<N>::kThreads, HalfCfg<N>::kMinBlocks)
    dst_half_kernel(const double* src, double* dst, int64_t nvec,
                    const double2* __restrict__ tw2, double scale, int64_t ld_src,
                    int64_t ld_dst, unsigned long long* ticket = nullptr) {
  using C = HalfCfg<N>;
  constexpr int V = C::V, T = C::T, F = C::F, n = N - 1;
  extern __shared__ __align__(16) double2 hbuf[];
  __shared__ double red[T > 32 ? 2 * (T / 32) : 2];
  const int f = F == 1 ? 0 : static_cast<int>(threadIdx.x) / T;
  const int t = F == 1 ? static_cast<int>(threadIdx.x) : static_cast<int>(threadIdx.x) % T;
  double2* fbuf = hbuf + f * C::kBuf;
  double* oa = reinterpret_cast<double*>(fbuf);
  double* ob = oa + opad<V>(N);
  const int64_t npairs = (nvec + 1) / 2;
  const int64_t nitems = (npairs + F - 1) / F;
  const double hs = 0.5 * scale;
  const int ldo = static_cast<int>(ld_dst);
  __shared__ int64_t s_next[2];
  int64_t item = blockIdx.x;
  if constexpr (DYN) {
    if (threadIdx.x == 0) s_next[1] = static_cast<int64_t>(atomicAdd(ticket, 1ull));
    __syncthreads();
    item = s_next[1];
  }
  for (int it = 0; item < nitems; ++it) {
    if constexpr (DYN) {
      if (threadIdx.x == 0) s_next[it & 1] = static_cast<int64_t>(atomicAdd(ticket, 1ull));
    }
    const int64_t g0 = 2 * (item * F + f);  // first vector of this FFT's pair
    const bool has_a = F == 1 || g0 < nvec, has_b = g0 + 1 < nvec;
    const double* sa = src + (has_a ? g0 : 0) * ld_src;
    const double* sb = has_b ? sa + ld_src : sa;
    double2 x[V];
#pragma unroll
    for (int p = 0; p < V; ++p) {
      const int m = t + T * p;
      x[p] = make_double2(0.0, 0.0);
      if (m > 0 && has_a) {
        const int mm = N - m;  // in 1..N-1 as well
        const double s = -__ldg(&tw2[m].y);
#ifdef STKG_DBG_NOLDG  // (measurement only: what the global loads cost)
        const double xb = double(m) * hs, xbm = double(mm) * hs;
        x[p] = half_pre(s, xb + 1.0, xbm - 1.0, xb, xbm);
#else
        const double xb = has_b ? sb[m - 1] : 0.0, xbm = has_b ? sb[mm - 1] : 0.0;
        x[p] = half_pre(s, sa[m - 1], sa[mm - 1], xb, xbm);
#endif
      }
    }
    if (STKG_DST_PREFETCH > 0 && !DYN) {  // a later item's 2F vectors into L2
      const int64_t nitem = item + STKG_DST_PREFETCH * int64_t(gridDim.x);
      if (nitem < nitems) {
        const int64_t nv0 = 2 * F * nitem;
        const int64_t nv = nvec - nv0 < 2 * F ? nvec - nv0 : 2 * F;
        const char* base = reinterpret_cast<const char*>(src + nv0 * ld_src);
        const int64_t bytes = nv * ld_src * int64_t(sizeof(double));
        for (int64_t o = int64_t(threadIdx.x) * 128; o < bytes; o += int64_t(C::kThreads) * 128)
          prefetch_l2(base + o);
      }
    }
    // (half_fft_post's first barrier orders these reads before fbuf is overwritten, and
    // the previous item's stores from fbuf before this item's first write: the trailing
    // __syncthreads below)
    half_fft_post<N, V, true>(x, fbuf, tw2, t, hs, red, OutSplit<V>{oa, ob});
    __syncthreads();
    if (STKG_DST_PREFETCH > 0 && DYN) {  // the next ticket's item into L2
      const int64_t nitem = s_next[it & 1];
      if (nitem < nitems) {
        const int64_t nv0 = 2 * F * nitem;
        const int64_t nv = nvec - nv0 < 2 * F ? nvec - nv0 : 2 * F;
        const char* base = reinterpret_cast<const char*>(src + nv0 * ld_src);
        const int64_t bytes = nv * ld_src * int64_t(sizeof(double));
        for (int64_t o = int64_t(threadIdx.x) * 128; o < bytes; o += int64_t(C::kThreads) * 128)
          prefetch_l2(base + o);
      }
    }
#ifdef STKG_DBG_NOSTG  // (measurement only: what the copy-out costs)
    if (hs == 123.456)
#endif
    if constexpr (F == 1) {
      double* da = dst + g0 * ld_dst;
      for (int e = t; e < ldo; e += T) da[e] = e < n ? oa[opad<V>(e)] : 0.0;
      if (has_b)
        for (int e = t; e < ldo; e += T) da[ld_dst + e] = e < n ? ob[opad<V>(e)] : 0.0;
    } else {
      // the item's vectors [2 item F, 2 item F + 2F) (back to back when ld_dst == n)
      const int64_t v0 = 2 * item * F;
      const int nv = static_cast<int>(nvec - v0 < 2 * F ? nvec - v0 : 2 * F);
      double* d0 = dst + v0 * ld_dst;
      for (int q = 0; q < nv; ++q) {  // vector q of the item (no division in the loop)
        const double* o_q = reinterpret_cast<const double*>(hbuf + (q >> 1) * C::kBuf) +
                            ((q & 1) ? opad<V>(N) : 0);
        for (int idx = threadIdx.x; idx < ldo; idx += C::kThreads)
          d0[int64_t(q) * ldo + idx] = idx < n ? o_q[opad<V>(idx)] : 0.0;
      }
      __syncthreads();  // other FFTs' buffers were read: next item may overwrite them
    }
    // (the barriers above ordered thread 0's ticket write of this iteration before this read;
    // the slot is rewritten two iterations later, after every thread has passed this read)
    if constexpr (DYN) {
      item = s_next[it & 1];
    } else {
      item += gridDim.x;
    }
  }
}

// Strided axis (inner > 1; element j of vector (o, i) at (o n + j) inner + i).  A tile is
// G = 2P neighbouring vectors (rows of 8G contiguous bytes), staged by cp.async; the P
// pairs run their FFTs side by side (P T threads, P T >= 128), each in its own shared
// region that holds first the two input rows, then the FFT, then the two output rows.
// Region pitch and row offsets are chosen so that the tile's row accesses are bank-conflict
// free.
template <int N>
struct HalfStridedCfg {
  static constexpr int V = half_v<N>(), T = N / V;
#ifdef STKG_HALF_P
  static constexpr int P = STKG_HALF_P;
#else
  static constexpr int P = T >= 32 ? 4 : 128 / T;
#endif
  static constexpr int G = 2 * P;
  static constexpr int kThreads = P * T;
  static constexpr int kMinBlocks = 65536 / (kThreads * 128) < 1 ? 1 : 65536 / (kThreads * 128);
  // Row v of the tile starts at (v/2) kRegion + (v%2) kRowB; with kStep = max(1, 16/G) these
  // are = kStep v (mod 16 doubles), so each half-warp's row accesses of 8 bytes hit distinct
  // banks.
#ifdef STKG_HALF_KSTEP
  static constexpr int kStep = STKG_HALF_KSTEP;
#else
  static constexpr int kStep = G >= 16 ? 1 : 16 / G;
#endif
  static constexpr int kRowB = N + N / V + kStep;                  // doubles: offset of row b
  static constexpr int kRegion = 2 * hpadded_len<N>() + 2 * kStep;  // doubles per pair
  static constexpr size_t kSmem = size_t(P) * kRegion * sizeof(double);
  static_assert(T <= 32 || T % 32 == 0, "FFTs are lane segments or whole warps");
};

template <int N>
__global__ void __launch_bounds__(HalfStridedCfg<N>::kThreads, HalfStridedCfg<N>::kMinBlocks)
    dst_half_strided_kernel(const double* src, double* dst, int64_t inner, int64_t nvec, const double2* __restrict__ tw2,
                            double scale) {
  using C = HalfStridedCfg<N>;
  constexpr int V = C::V, T = C::T, P = C::P, G = C::G, n = N - 1;
  constexpr int RB = C::kRowB, RG = C::kRegion;
  extern __shared__ __align__(16) double smem[];
  __shared__ int64_t vbase[G];
  __shared__ double red[P][T > 32 ? 2 * (T / 32) : 2];
  const int f = threadIdx.x / T, t = threadIdx.x % T;
  double* region = smem + f * RG;
  double2* fbuf = reinterpret_cast<double2*>(region);
  const int64_t ntiles = (nvec + G - 1) / G;
  const double hs = 0.5 * scale;
  auto row = [&](int v) { return smem + (v >> 1) * RG + (v & 1) * RB; };
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    __syncthreads();  // the previous tile's stores have read the staging rows
    for (int v = threadIdx.x; v < G; v += C::kThreads) {
      const int64_t g = tile * G + v;
      vbase[v] = g < nvec ? (g / inner) * n * inner + g % inner : -1;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < G * n; e += C::kThreads) {
      const int v = e % G, jj = e / G;
      const int64_t b = vbase[v];
      cp_async8(row(v) + jj, b >= 0 ? src + b + int64_t(jj) * inner : src, b >= 0);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    const double* ra = region;
    const double* rb = region + RB;
    double2 x[V];
#pragma unroll
    for (int p = 0; p < V; ++p) {
      const int m = t + T * p;
      x[p] = make_double2(0.0, 0.0);
      if (m > 0) {
        const int mm = N - m;
        const double s = -__ldg(&tw2[m].y);
        x[p] = half_pre(s, ra[m - 1], ra[mm - 1], rb[m - 1], rb[mm - 1]);
      }
    }
    half_fft_post<N, V>(x, fbuf, tw2, t, hs, red[f], OutSplit<V>{region, region + RB},
                        P > 1 ? 1 + f : 0);
    __syncthreads();
    for (int e = threadIdx.x; e < G * n; e += C::kThreads) {
      const int v = e % G, kk = e / G;
      const int64_t b = vbase[v];
      if (b >= 0) __stcs(dst + b + int64_t(kk) * inner, row(v)[opad<V>(kk)]);
    }
  }
}


__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

// Strided axis, 16-byte variant for the padded internal layout of heat.cu's device solve
// (fastest axis stored with pitch N = n + 1, so inner is a multiple of the tile width G and
// every tile row is 16P-byte aligned).  The tile is staged by 16-byte cp.async into a
// mirror of its global rows (row r = P chunks of 16 bytes, chunk c = the values (a_r, b_r)
// of pair c), XOR-swizzled within the row -- the layout TMA's SWIZZLE_64B/128B modes
// produce: cp.async coalesces a global row only when its shared destination is the same
// contiguous segment (tools/microbench/ldgsts_probe.cu: 1.5x the L2 sectors and 1.8x the
// time for the per-pair-region layout), and the swizzle makes the pre-processing's
// reads of 8 consecutive rows of one pair conflict-free.  After every pair has read its
// inputs (a CTA barrier), the tile space is reused by the pairs' FFT regions; the outputs
// (OutPair) leave as 16-byte streaming stores.  In place is allowed (src == dst): a tile
// is read completely before it is written.
// Default pairs per tile: 4 (64-byte rows) for FFTs of whole warps, else 128 threads.
#ifndef STKG_HALF2_V
#define STKG_HALF2_V STKG_HALF_V
#endif
// Values per thread of the strided kernel's FFTs (tuning knob STKG_HALF2_V; falls back to
// half_v when the FFT would not span whole warps).
template <int N>
constexpr int half2_v() { return N / STKG_HALF2_V >= 32 ? STKG_HALF2_V : half_v<N>(); }
template <int N>
constexpr int half2_pairs() { return N / half2_v<N>() >= 32 ? 4 : 128 / (N / half2_v<N>()); }

// PF (prefetch): the staged tile gets its own buffer beside the pair regions, and the next
// tile's copy is issued as soon as every pair has read the current one, so it lands while
// the FFTs run (more shared memory per CTA, fewer CTAs per SM).
template <int N, int PP = half2_pairs<N>(), bool PF = false>
struct HalfStrided2Cfg {
  static constexpr int V = half2_v<N>(), T = N / V;
  static constexpr int P = PP;       // vector pairs per tile
  static constexpr int G = 2 * P;    // vectors per tile
  static constexpr int kThreads = P * T;
#ifdef STKG_HALF2_MINB
  static constexpr int kMinBlocks = STKG_HALF2_MINB;
#else
  static constexpr int kMinBlocks = 65536 / (kThreads * 128) < 1 ? 1 : 65536 / (kThreads * 128);
#endif
  // double2 per pair region (FFT, outputs), rounded to 128 bytes plus a skew: the output
  // copy interleaves the P regions (q = e % P), so consecutive regions start 8/P (P <= 4) or
  // 1 (P >= 8) 16-byte bank groups apart and every quarter-warp phase of 8 16-byte reads
  // hits 8 distinct groups
  static constexpr int kRegion = (hpadded_len<N>() + 7) / 8 * 8 + (P >= 8 ? 1 : 8 / P);
  static constexpr int kTile = ((N - 1) * P + 7) / 8 * 8;  // double2 of the staged tile
  static constexpr int kTileOff = PF ? P * kRegion : 0;   // where the tile is staged
  static constexpr int kSmemD2 = PF ? P * kRegion + kTile
                                    : (P * kRegion > kTile ? P * kRegion : kTile);
  static constexpr size_t kSmem = size_t(kSmemD2) * sizeof(double2);
  static_assert(T <= 32 || T % 32 == 0, "FFTs are lane segments or whole warps");
  static_assert(P == 1 || P == 2 || P == 4 || P % 8 == 0, "tile rows of 16, 32, 64 or 128k bytes");
  static_assert(N - 1 + (N - 2) / 16 < kRegion && N <= kRegion, "OutPair staging fits the region");
  // 16-byte chunk of pair c in tile row r, XOR-swizzled so that 8 consecutive rows of one
  // pair fall in 8 distinct 16-byte bank groups (SWIZZLE_32B/64B/128B-like)
  __device__ __forceinline__ static int chunk(int r, int c) {
    if constexpr (P == 1) return c;  // 16-byte rows: consecutive rows are distinct groups
    else if constexpr (P == 2) return c ^ ((r >> 2) & 1);
    else if constexpr (P == 4) return c ^ ((r >> 1) & 3);
    else return c ^ (r & 7);
  }
};

template <int N, int PP = half2_pairs<N>(), bool PF = false>
__global__ void __launch_bounds__(HalfStrided2Cfg<N, PP, PF>::kThreads,
                                  HalfStrided2Cfg<N, PP, PF>::kMinBlocks)
    dst_half_strided2_kernel(const double* src, double* dst, int64_t inner, int64_t nvec,
                             const double2* __restrict__ tw2, double scale) {
  using C = HalfStrided2Cfg<N, PP, PF>;
  constexpr int V = C::V, T = C::T, P = C::P, G = C::G, n = N - 1, RG = C::kRegion;
  extern __shared__ __align__(128) double2 sreg[];
  __shared__ double red[P][T > 32 ? 2 * (T / 32) : 2];
  const int f = threadIdx.x / T, t = threadIdx.x % T;
  double2* region = sreg + f * RG;
  double2* stile = sreg + C::kTileOff;
  const int64_t ntiles = nvec / G;  // the host guarantees inner % G == 0
  const double hs = 0.5 * scale;
  auto tile_base = [&](int64_t tile) {
    const int64_t g = tile * G;
    return (g / inner) * n * inner + g % inner;
  };
  auto load_tile = [&](int64_t base) {
    for (int e = threadIdx.x; e < P * n; e += C::kThreads) {
      const int c = e % P, r = e / P;
      cp_async16(stile + r * P + C::chunk(r, c), src + base + int64_t(r) * inner + 2 * c);
    }
    cp_async_commit();
  };
  if (PF && blockIdx.x < ntiles) load_tile(tile_base(blockIdx.x));
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile_base(tile);
    if (!PF) {
      __syncthreads();  // the previous tile's stores have read the regions
      load_tile(base);
    }
    cp_async_wait<0>();
    __syncthreads();  // (PF: also orders the previous tile's stores before the FFT writes)
    double2 x[V];
#pragma unroll
    for (int p = 0; p < V; ++p) {
      const int m = t + T * p;
      x[p] = make_double2(0.0, 0.0);
      if (m > 0) {
        const int r0 = m - 1, r1 = N - m - 1;
        const double s = -__ldg(&tw2[m].y);
        const double2 u = stile[r0 * P + C::chunk(r0, f)], w = stile[r1 * P + C::chunk(r1, f)];
        x[p] = half_pre(s, u.x, w.x, u.y, w.y);
      }
    }
    __syncthreads();  // every pair has read the tile: the regions / the next tile may overwrite it
    if (PF && tile + gridDim.x < ntiles) load_tile(tile_base(tile + gridDim.x));

    half_fft_post<N, V>(x, region, tw2, t, hs, red[f], OutPair<N>{region}, P > 1 ? 1 + f : 0);
    __syncthreads();
    for (int e = threadIdx.x; e < P * n; e += C::kThreads) {
      const int q = e % P, kk = e / P;
      __stcs(reinterpret_cast<double2*>(dst + base + int64_t(kk) * inner + 2 * q),
             sreg[q * RG + OutPair<N>::idx(kk)]);
    }
  }
}

// ---------------------------------------------------------------------------------------
// Strided axis, TMA variant of dst_half_strided2_kernel for tiles of 4 pairs (64-byte rows,
// N = 512, 1024): one thread arms an mbarrier and issues the tile as ceil(n / 256) 2D TMA
// boxes of {8 doubles, 256 rows} with SWIZZLE_64B, which lands exactly the swizzled row
// mirror the pre-processing reads (16-byte chunk c of row r at c ^ ((r >> 1) & 3)).  The
// copy leaves the LSU pipe: no per-thread cp.async instructions, address arithmetic or
// shared-memory store wavefronts.  The tensor map views the buffer as [outer * n rows] x
// [inner columns] (row stride inner * 8 bytes); the last box's extra rows read the next
// block's first rows (or are zero-filled past the end) and are never used.
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load_1d(void* smem, const void* gmem, unsigned bytes,
                                             uint64_t* bar) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(s),
      "l"(gmem), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(s),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(b)
      : "memory");
}

template <int N>
struct HalfStridedTmaCfg {
  using B = HalfStrided2Cfg<N, 4, false>;
#ifdef STKG_TMA_BOX
  static constexpr int kBoxRows = STKG_TMA_BOX;
#else
  static constexpr int kBoxRows = 256;
#endif
  static constexpr int kBoxes = (N - 1 + kBoxRows - 1) / kBoxRows;
  static constexpr int kTileBytes = kBoxes * kBoxRows * 64;
  static constexpr size_t kRegionsBytes = size_t(B::P) * B::kRegion * sizeof(double2);
  // + 512 bytes so the tile can be aligned to the 512-byte SWIZZLE_64B pattern
  static constexpr size_t kSmem =
      (kRegionsBytes > size_t(kTileBytes) ? kRegionsBytes : size_t(kTileBytes)) + 512;
  static_assert(B::T >= 32, "TMA variant: tiles of 4 pairs (whole-warp FFTs)");
};

template <int N>
__global__ void __launch_bounds__(HalfStrided2Cfg<N, 4, false>::kThreads,
                                  HalfStrided2Cfg<N, 4, false>::kMinBlocks)
    dst_half_strided_tma_kernel(const __grid_constant__ CUtensorMap map, double* dst,
                                int64_t inner, int64_t nvec, const double2* __restrict__ tw2,
                                double scale) {
  using C = HalfStrided2Cfg<N, 4, false>;
  using TC = HalfStridedTmaCfg<N>;
  constexpr int V = C::V, T = C::T, P = C::P, G = C::G, n = N - 1, RG = C::kRegion;
  extern __shared__ __align__(128) unsigned char sraw[];
  double2* sreg = reinterpret_cast<double2*>(
      (reinterpret_cast<uintptr_t>(sraw) + 511) & ~uintptr_t(511));
  __shared__ double red[P][T > 32 ? 2 * (T / 32) : 2];
  __shared__ __align__(8) uint64_t bar;
  const int f = threadIdx.x / T, t = threadIdx.x % T;
  double2* region = sreg + f * RG;
  const int64_t ntiles = nvec / G;  // the host guarantees inner % G == 0
  const double hs = 0.5 * scale;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  unsigned phase = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t g = tile * G;
    const int64_t o = g / inner, i0 = g - o * inner;
    const int64_t base = o * n * inner + i0;
    __syncthreads();  // the previous tile's stores have read the regions (and bar is set up)
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_arrive_expect_tx(&bar, TC::kTileBytes);
#pragma unroll
      for (int b = 0; b < TC::kBoxes; ++b)
        tma_load_2d(reinterpret_cast<char*>(sreg) + b * TC::kBoxRows * 64, &map,
                    static_cast<int>(i0), static_cast<int>(o * n + b * TC::kBoxRows), &bar);
    }
    mbar_wait(&bar, phase);
    phase ^= 1u;
    double2 x[V];
#pragma unroll
    for (int p = 0; p < V; ++p) {
      const int m = t + T * p;
      x[p] = make_double2(0.0, 0.0);
      if (m > 0) {
        const int r0 = m - 1, r1 = N - m - 1;
        const double s = -__ldg(&tw2[m].y);
        const double2 u = sreg[r0 * P + C::chunk(r0, f)], w = sreg[r1 * P + C::chunk(r1, f)];
        x[p] = half_pre(s, u.x, w.x, u.y, w.y);
      }
    }
    __syncthreads();  // every pair has read the tile: the regions may overwrite it
    half_fft_post<N, V>(x, region, tw2, t, hs, red[f], OutPair<N>{region}, 1 + f);
    __syncthreads();
    for (int e = threadIdx.x; e < P * n; e += C::kThreads) {
      const int q = e % P, kk = e / P;
      __stcs(reinterpret_cast<double2*>(dst + base + int64_t(kk) * inner + 2 * q),
             sreg[q * RG + OutPair<N>::idx(kk)]);
    }
  }
}

// Contiguous axis, bulk-copy input (one vector pair per CTA, T >= 64): the pair's two vectors
// are one contiguous, 16-byte aligned region of the source (pairs start at even vectors), so
// a single cp.async.bulk brings them into the FFT buffer and the pre-processing reads shared
// memory instead of issuing 4 V global loads per thread against rows that are only 8-byte
// aligned.  A later item is prefetched into L2 as in dst_half_kernel.  The last vector of an
// odd count keeps the per-thread loads.
// SEP (measurement variant, off): the pair lands in its own buffer behind the FFT buffer
// (16 N more bytes per CTA, 6 instead of 8 CTAs per SM), and the next item's copy is issued as
// soon as this item's inputs are in registers, so it lands while the FFT and the copy-out
// run.  Measured slower (cfg3 11.08 vs 10.38 ms): the lost occupancy costs more than the
// overlap inside one CTA gains -- the other CTAs of the SM already cover the landing time.
#ifndef STKG_DST_BULK_SEP
#define STKG_DST_BULK_SEP 0
#endif
template <int N, bool SEP = (STKG_DST_BULK_SEP != 0)>
__global__ void __launch_bounds__(HalfCfg<N>::kThreads, SEP ? 6 : HalfCfg<N>::kMinBlocks)
    dst_half_bulk_kernel(const double* src, double* dst, int64_t nvec,
                         const double2* __restrict__ tw2, double scale, int64_t ld_src,
                         int64_t ld_dst) {
  using C = HalfCfg<N>;
  constexpr int V = C::V, T = C::T, n = N - 1;
  static_assert(C::F == 1, "one pair per CTA");
  extern __shared__ __align__(16) double2 hbuf[];
  __shared__ double red[T > 32 ? 2 * (T / 32) : 2];
  __shared__ __align__(8) uint64_t bar;
  const int t = static_cast<int>(threadIdx.x);
  double2* fbuf = hbuf;
  double* oa = reinterpret_cast<double*>(fbuf);
  double* ob = oa + opad<V>(N);
  // the landed pair, linear
  const double* lin = reinterpret_cast<const double*>(SEP ? hbuf + C::kBuf : fbuf);
  const int64_t nitems = (nvec + 1) / 2;
  const double hs = 0.5 * scale;
  const int ldo = static_cast<int>(ld_dst), ldi = static_cast<int>(ld_src);
  if (t == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned phase = 0;
  auto issue = [&](int64_t it) {  // thread 0: the pair of item `it` (complete pairs only)
    const unsigned bytes = static_cast<unsigned>(2 * ld_src * sizeof(double));
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    mbar_arrive_expect_tx(&bar, bytes);
    bulk_load_1d(const_cast<double*>(lin), src + 2 * it * ld_src, bytes, &bar);
  };
  if (SEP && t == 0 && int64_t(blockIdx.x) < nitems && 2 * int64_t(blockIdx.x) + 1 < nvec)
    issue(blockIdx.x);
  for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int64_t g0 = 2 * item;
    const bool has_b = g0 + 1 < nvec;
    const double* sa = src + g0 * ld_src;
    double2 x[V];
    if (has_b) {
      if (!SEP && t == 0) issue(item);
      if (STKG_DST_PREFETCH > 0) {  // a later item's pair into L2 while this one lands
        const int64_t nitem = item + STKG_DST_PREFETCH * int64_t(gridDim.x);
        if (nitem < nitems) {
          const char* base = reinterpret_cast<const char*>(src + 2 * nitem * ld_src);
          const int64_t bytes = (nvec - 2 * nitem < 2 ? 1 : 2) * ld_src * int64_t(sizeof(double));
          for (int64_t o = int64_t(t) * 128; o < bytes; o += int64_t(C::kThreads) * 128)
            prefetch_l2(base + o);
        }
      }
      mbar_wait(&bar, phase);
      phase ^= 1u;
#pragma unroll
      for (int p = 0; p < V; ++p) {
        const int m = t + T * p;
        x[p] = make_double2(0.0, 0.0);
        if (m > 0) {
          const int mm = N - m;
          const double s = -__ldg(&tw2[m].y);
          x[p] = half_pre(s, lin[m - 1], lin[mm - 1], lin[ldi + m - 1], lin[ldi + mm - 1]);
        }
      }
      if constexpr (SEP) {
        __syncthreads();  // every thread holds its inputs: the next pair may land
        const int64_t nx = item + gridDim.x;
        if (t == 0 && nx < nitems && 2 * nx + 1 < nvec) issue(nx);
      }
    } else {
#pragma unroll
      for (int p = 0; p < V; ++p) {
        const int m = t + T * p;
        x[p] = make_double2(0.0, 0.0);
        if (m > 0) {
          const double s = -__ldg(&tw2[m].y);
          x[p] = half_pre(s, sa[m - 1], sa[N - m - 1], 0.0, 0.0);
        }
      }
    }
    // (half_fft_post's first barrier orders the reads of the landed pair before fbuf is
    // overwritten by the first stage)
    half_fft_post<N, V, true>(x, fbuf, tw2, t, hs, red, OutSplit<V>{oa, ob});
    __syncthreads();
    double* da = dst + g0 * ld_dst;
    for (int e = t; e < ldo; e += T) da[e] = e < n ? oa[opad<V>(e)] : 0.0;
    if (has_b)
      for (int e = t; e < ldo; e += T) da[ld_dst + e] = e < n ? ob[opad<V>(e)] : 0.0;
    __syncthreads();  // the staging was read: the next pair may land in fbuf
  }
}

}  // namespace stkg
