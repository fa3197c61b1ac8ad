// Shared-memory wavefronts of cp.async (LDGSTS) tile copies for the strided DST pass.
// A tile = 1023 rows of 64 contiguous bytes (8 doubles = 4 vector pairs), row stride
// 8192 bytes (the padded cfg3 layout).  Each pattern copies every tile of a 64-slice
// buffer into shared memory with a different thread -> (row, chunk) map or shared layout;
// run under ncu with l1tex__data_pipe_lsu_wavefronts_mem_shared.sum to compare.
//   A: 16 B, q = e % 4, row = e / 4, dst = region q (1090 double2 apart) + row
//   B: 16 B, same map, dst = row * 4 + q (mirror of the global rows, 64 B pitch)
//   C: 16 B, same map, dst = row * 5 + q (80 B pitch)
//   D: 16 B, q = e / 1023, row = e % 1023 (a warp copies one pair's column), dst = region q + row
//   F: 16 B, as B with the 16-byte chunks XOR-swizzled by (row >> 1) & 3 (TMA SWIZZLE_64B)
//   E:  8 B, v = e % 8, row = e / 8, dst = per-vector rows (the unpadded kernel's pattern)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int n = 1023, RG = 1090;

__device__ __forceinline__ void cp16(void* s, const void* g) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(g));
}
__device__ __forceinline__ void cp8(void* s, const void* g) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(a), "l"(g));
}

template <int PAT>
__global__ void __launch_bounds__(256) probe(const double* src, double* sink, int64_t ntiles) {
  extern __shared__ __align__(16) double2 sm[];
  double acc = 0.0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = (tile / 128) * int64_t(n) * 1024 + (tile % 128) * 8;
    __syncthreads();
    for (int e = threadIdx.x; e < 4 * n; e += 256) {
      if (PAT == 0) cp16(sm + (e % 4) * RG + e / 4, src + base + int64_t(e / 4) * 1024 + 2 * (e % 4));
      if (PAT == 1) cp16(sm + (e / 4) * 4 + e % 4, src + base + int64_t(e / 4) * 1024 + 2 * (e % 4));
      if (PAT == 2) cp16(sm + (e / 4) * 5 + e % 4, src + base + int64_t(e / 4) * 1024 + 2 * (e % 4));
      if (PAT == 5) {  // F: mirror rows with the 64-byte XOR swizzle (TMA SWIZZLE_64B layout)
        const int r = e / 4, c = e % 4;
        cp16(sm + r * 4 + (c ^ ((r >> 1) & 3)), src + base + int64_t(r) * 1024 + 2 * c);
      }
      if (PAT == 3) cp16(sm + (e / n) * RG + e % n, src + base + int64_t(e % n) * 1024 + 2 * (e / n));
    }
    if (PAT == 4) {
      double* d = reinterpret_cast<double*>(sm);
      for (int e = threadIdx.x; e < 8 * n; e += 256)
        cp8(d + (e % 8) * 1100 + e / 8, src + base + int64_t(e / 8) * 1024 + e % 8);
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
    __syncthreads();
    acc += reinterpret_cast<const double*>(sm)[threadIdx.x];
  }
  if (acc == 12345.0) sink[0] = acc;
}

int main() {
  const int64_t nt = 64, elems = nt * n * 1024, ntiles = nt * 128;
  double *src, *sink;
  cudaMalloc(&src, elems * 8);
  cudaMalloc(&sink, 8);
  cudaMemset(src, 0, elems * 8);
  const int smem = 92 * 1024;
  auto run = [&](auto k, const char* name) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<<<296, 256, smem>>>(src, sink, ntiles);
    cudaEventRecord(a);
    k<<<296, 256, smem>>>(src, sink, ntiles);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("%s %.1f us  %.0f GB/s\n", name, 1e3 * ms, elems * 8 / (ms * 1e6));
  };
  run(probe<0>, "A region-skew 16B");
  run(probe<1>, "B mirror-64B   16B");
  run(probe<2>, "C pitch-80B    16B");
  run(probe<3>, "D column/warp  16B");
  run(probe<4>, "E per-vector    8B");
  run(probe<5>, "F mirror-swz64 16B");
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
