// Throughput of the legacy warp-level INT8 tensor-core MMA (mma.sync m16n8k32 s8 -> s32) on
// sm_100a, registers only: is it fast enough for an INT8-sliced (Ozaki) FP64 GEMM?
#include <cstdio>
#include <cstdint>

__global__ void imma_loop(int* out, int iters) {
  int a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  int c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  int s = 0;
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x, b = a + 1;
  double c[8][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int* o;
  double* od;
  cudaMalloc(&o, 148 * 8 * 256 * 4);
  cudaMalloc(&od, 148 * 8 * 256 * 8);
  const int iters = 4096, blocks = 148 * 4, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  imma_loop<<<blocks, threads>>>(o, 16);
  cudaEventRecord(e0);
  imma_loop<<<blocks, threads>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * 16 * 8 * 32 * 8.0 * iters * (blocks * threads / 32.0);
  printf("IMMA m16n8k32 s8: %.1f TOPS\n", ops / ms / 1e9);
  dmma_loop<<<blocks, threads>>>(od, 16);
  cudaEventRecord(e0);
  dmma_loop<<<blocks, threads>>>(od, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (blocks * threads / 32.0);
  printf("DMMA m8n8k4 f64:  %.1f TFLOPS\n", flops / ms / 1e9);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
