// Shared infrastructure for the stk_gpu C ABI: status codes, thread-local error text,
// CUDA error mapping, deterministic reductions and the counter-based generator.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/stk_gpu.h"

namespace stkg {

// Exceptions inside the library carry the status code of the reference exception class
// they stand for (stk/errors.hpp:9-42); the C ABI converts them back into codes.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_error(const std::string& msg);

#define STKG_CUDA_CHECK(expr)                                                             \
  do {                                                                                    \
    cudaError_t err__ = (expr);                                                           \
    if (err__ != cudaSuccess)                                                             \
      throw ::stkg::Error(STKG_CUDA, std::string(#expr) + ": " + cudaGetErrorString(err__) + \
                                         " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

#define STKG_REQUIRE(cond, code, msg)             \
  do {                                            \
    if (!(cond)) throw ::stkg::Error(code, msg);  \
  } while (0)

// Run a body, translate exceptions into status codes + thread-local message.
template <typename F>
int guarded(F&& body) {
  try {
    body();
    return STKG_OK;
  } catch (const Error& e) {
    set_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return STKG_CUDA;
  } catch (const std::exception& e) {
    set_error(e.what());
    return STKG_NUMERIC;
  }
}

// Device buffer owning RAII wrapper.
struct DevBuf {
  double* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    release();
    if (count) STKG_CUDA_CHECK(cudaMalloc(&p, count * sizeof(double)));
    n = count;
  }
  void upload(const double* host, size_t count, cudaStream_t s) {
    STKG_CUDA_CHECK(cudaMemcpyAsync(p, host, count * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// ---------------------------------------------------------------- reductions ------
// Deterministic two-level sum: a fixed grid of kReduceBlocks partial sums, each block a
// fixed-order tree; the partials are then summed in index order by one block.  Same
// inputs + same sizes => bit-identical result.
// The grid is a fixed constant (not derived from the SM count) so that results do not
// depend on the device the reduction runs on.
constexpr int kReduceBlocks = 592;
constexpr int kReduceThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of v (all threads must call); result valid in thread 0.
template <int THREADS>
__device__ __forceinline__ double block_sum(double v, double* smem /* >= THREADS/32 */) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < THREADS / 32 ? smem[lane] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------- generator -------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ double uniform_pm1(uint64_t seed, uint64_t stream,
                                                       uint64_t index) {
  const uint64_t x = splitmix64(seed ^ (stream << 40) ^ index);
  const double u = (double)(x >> 11) * 0x1.0p-53;
  return 2.0 * u - 1.0;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Multiprocessor count of the current device (148 on B200), queried once per device.
inline int num_sms() {
  static thread_local int cached_dev = -1, cached_sms = 0;
  int dev = 0;
  STKG_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev != cached_dev) {
    STKG_CUDA_CHECK(cudaDeviceGetAttribute(&cached_sms, cudaDevAttrMultiProcessorCount, dev));
    cached_dev = dev;
  }
  return cached_sms;
}

}  // namespace stkg
