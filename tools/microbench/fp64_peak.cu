// FP64 pipe microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync f64 shapes).
// Measures the FP64 roofline denominator that MEASURED_PEAKS.json lacks.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

// m8n8k4: A 1 f64, B 1 f64, C/D 2 f64 per thread
__global__ void dmma_m8n8k4_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// m16n8k4: A 2 f64, B 1, C 4
__global__ void dmma_m16n8k4_kernel(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-12, a1 = 0.25, b = 0.5;
  double c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

// m16n8k16: A 8 f64, B 4, C 4
__global__ void dmma_m16n8k16_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + i * 1e-3 + threadIdx.x * 1e-12;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 0.5 + i * 1e-3;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

template <typename F>
float time_it(F launch, int reps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main() {
  double* out; CK(cudaMalloc(&out, 8));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  const int iters = 4096;
  for (int tpb : {256, 512}) for (int bps : {2, 4, 8}) {
    int blocks = sms * bps;
    float ms = time_it([&] { dfma_kernel<8><<<blocks, tpb>>>(out, iters, 1.0000001, 1e-7); }, 5);
    double flops = 2.0 * 8 * iters * (double)blocks * tpb;
    printf("DFMA  tpb %d blocks/SM %d : %.2f TFLOP/s (%.3f ms)\n", tpb, bps, flops / ms / 1e9, ms);
  }
  for (int tpb : {128, 256, 512}) for (int bps : {1, 2, 4}) {
    int blocks = sms * bps;
    float ms = time_it([&] { dmma_m8n8k4_kernel<<<blocks, tpb>>>(out, iters); }, 5);
    double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (tpb / 32);
    printf("DMMA m8n8k4   tpb %d blocks/SM %d : %.2f TFLOP/s\n", tpb, bps, flops / ms / 1e9);
    ms = time_it([&] { dmma_m16n8k4_kernel<<<blocks, tpb>>>(out, iters); }, 5);
    flops = 2.0 * 16 * 8 * 4 * 8 * (double)iters * blocks * (tpb / 32);
    printf("DMMA m16n8k4  tpb %d blocks/SM %d : %.2f TFLOP/s\n", tpb, bps, flops / ms / 1e9);
    ms = time_it([&] { dmma_m16n8k16_kernel<<<blocks, tpb>>>(out, iters / 4); }, 5);
    flops = 2.0 * 16 * 8 * 16 * 4 * (double)(iters / 4) * blocks * (tpb / 32);
    printf("DMMA m16n8k16 tpb %d blocks/SM %d : %.2f TFLOP/s\n", tpb, bps, flops / ms / 1e9);
  }
  CK(cudaGetLastError());
  // sustained: DMMA m16n8k16 for ~4 s
  {
    int blocks = sms * 2, tpb = 256;
    int it = 1 << 16;
    float ms = time_it([&] { dmma_m16n8k16_kernel<<<blocks, tpb>>>(out, it); }, 3);
    double flops = 2.0 * 16 * 8 * 16 * 4 * (double)it * blocks * (tpb / 32);
    printf("DMMA m16n8k16 sustained (%.1f ms/launch): %.2f TFLOP/s\n", ms, flops / ms / 1e9);
    ms = time_it([&] { dfma_kernel<8><<<blocks*2, 256>>>(out, it * 4, 1.0000001, 1e-7); }, 3);
    flops = 2.0 * 8 * it * 4.0 * blocks * 2 * 256;
    printf("DFMA sustained (%.1f ms/launch): %.2f TFLOP/s\n", ms, flops / ms / 1e9);
  }
  return 0;
}
