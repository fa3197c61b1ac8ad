// Standalone timing of the half-length DST kernels on the cfg3 geometry (64 slices):
// contiguous and strided passes on device-resident data (a rotating variant was measured
// here too: 0.480 ms vs 0.395 strided and 0.267 contiguous; see DESIGN K2b).
#include <cstdio>
#include <cmath>
#include <vector>
#include "dst_half.cuh"
using namespace stkg;

template <class K>
float time_it(K launch, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  constexpr int N = 1024, n = N - 1;
  const int64_t B = 64, R = n, nvec = B * R;
  const size_t count = size_t(B) * n * n;
  double *src, *dst;
  double2* tw;
  cudaMalloc(&src, count * 8);
  cudaMalloc(&dst, count * 8);
  cudaMalloc(&tw, 2 * N * sizeof(double2));
  std::vector<double2> h(2 * N);
  for (int m = 0; m < 2 * N; ++m) h[m] = make_double2(cos(M_PI * m / N), -sin(M_PI * m / N));
  cudaMemcpy(tw, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice);
  cudaMemset(src, 0, count * 8);
  const double scale = sqrt(2.0 / N);
  int pc = 0, ps = 0;
  cudaFuncSetAttribute(dst_half_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HalfCfg<N>::kSmem);
  cudaFuncSetAttribute(dst_half_strided_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HalfStridedCfg<N>::kSmem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pc, dst_half_kernel<N>, HalfCfg<N>::kThreads, HalfCfg<N>::kSmem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, dst_half_strided_kernel<N>, HalfStridedCfg<N>::kThreads, HalfStridedCfg<N>::kSmem);
  auto contig = [&] {
    dst_half_kernel<N><<<148 * pc, HalfCfg<N>::kThreads, HalfCfg<N>::kSmem>>>(src, dst, nvec, tw, scale);
  };
  auto strided = [&] {  // x-axis of [B][n][n]: inner = n, outer = B
    dst_half_strided_kernel<N><<<148 * ps, HalfStridedCfg<N>::kThreads, HalfStridedCfg<N>::kSmem>>>(src, dst, R, nvec, tw, scale);
  };
  const double gb = 16.0 * count / 1e9;
  float tc = time_it(contig, 10), ts = time_it(strided, 10);
  printf("occupancy (CTAs/SM): contig %d strided %d\n", pc, ps);
  printf("contiguous %.3f ms (%.0f GB/s)\nstrided    %.3f ms (%.0f GB/s)\n", tc, gb / tc * 1e3, ts,
         gb / ts * 1e3);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
