// Config sweep for the FP64 DMMA GEMM (paper_1912_10082_b200/csrc/gemm_f64.cuh) on the heat
// transform shapes and the wave preconditioner shape.  Dev tool; not part of the product.
#include <cstdio>
#include <vector>
#include "../../paper_1912_10082_b200/csrc/gemm_f64.cuh"

using namespace stkg;
namespace stkg { void set_error(const std::string&) {} }

using C1 = GemmCfg<128, 128, 16, 64, 32, 4, 1>;
using C9 = GemmCfg<128, 64, 16, 64, 32, 3, 2>;
using C10 = GemmCfg<128, 64, 32, 64, 32, 2, 2>;
using C11 = GemmCfg<128, 64, 16, 64, 32, 4, 2>;
using C5 = GemmCfg<64, 64, 16, 32, 32, 4, 3>;
using C12 = GemmCfg<64, 64, 16, 32, 32, 3, 3>;
using C13 = GemmCfg<64, 128, 16, 32, 64, 3, 2>;
using C14 = GemmCfg<64, 64, 32, 32, 32, 2, 3>;
using C15 = GemmCfg<32, 64, 32, 32, 32, 2, 4>;
using C16 = GemmCfg<64, 32, 32, 32, 32, 2, 4>;
using C17 = GemmCfg<32, 32, 32, 32, 32, 2, 8>;
using C18 = GemmCfg<64, 64, 16, 32, 32, 3, 3>;
using C19 = GemmCfg<64, 64, 32, 32, 16, 2, 2>;  // 8 warps of 32x16
using C20 = GemmCfg<64, 64, 32, 16, 32, 2, 2>;  // 8 warps of 16x32
using C21 = GemmCfg<64, 64, 32, 32, 16, 3, 2>;  // 8 warps, 3 stages
using C22 = GemmCfg<48, 64, 48, 16, 32, 2, 3>;  // 48-row tiles: 374 tiles at the 1k shape
template <class Cfg>
float run(const GemmProblem& p, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch_gemm_cfg<Cfg>(p, EpiStore{}, 0);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) launch_gemm_cfg<Cfg>(p, EpiStore{}, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

__global__ void fill(double* x, size_t n, unsigned s) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    x[i] = double((i * 2654435761u + s) % 1000003) / 1000003.0 - 0.5;
}

__global__ void maxdiff(const double* a, const double* b, size_t n, double* out) {
  double m = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(a[i] - b[i]));
  atomicMax((unsigned long long*)out, __double_as_longlong(m));
}

int main() {
  const int64_t n = 1023, nt = 64;
  const size_t big = n * n * nt;
  double *X, *F, *C, *Cref, *d;
  cudaMalloc(&X, n * n * 8);
  cudaMalloc(&F, big * 8);
  cudaMalloc(&C, big * 8);
  cudaMalloc(&Cref, big * 8);
  cudaMalloc(&d, 8);
  fill<<<1024, 256>>>(X, n * n, 1);
  fill<<<1024, 256>>>(F, big, 7);
  struct Shape { const char* name; GemmProblem p; };
  std::vector<Shape> shapes;
  {
    GemmProblem p; p.M = n; p.K = n; p.N = n * nt; p.A = X; p.lda = n; p.B = F; p.ldb = n; p.C = C; p.ldc = n;
    shapes.push_back({"left  1023x1023 * 1023x65472", p});
  }
  {
    GemmProblem p; p.M = n; p.K = n; p.N = n; p.batch = nt; p.A = F; p.lda = n; p.strideA = n * n;
    p.B = X; p.ldb = n; p.C = C; p.ldc = n; p.strideC = n * n;
    shapes.push_back({"right 64 x (1023x1023 * 1023x1023)", p});
  }
  {
    GemmProblem p; p.M = n; p.K = n; p.N = 1025; p.A = X; p.lda = n; p.B = F; p.ldb = n; p.C = C; p.ldc = n;
    shapes.push_back({"single 1023x1023 * 1023x1025", p});
  }
  for (int ks : {2, 3, 4}) {  // split-K emulation: ks K-slices of the single shape as a batch
    GemmProblem p; p.M = n; p.K = (n + ks - 1) / ks; p.N = 1025; p.batch = ks; p.A = X; p.lda = n;
    p.strideA = p.K * n; p.B = F; p.ldb = n; p.strideB = p.K; p.C = C; p.ldc = n;
    p.strideC = n * 1025;
    static char names[3][64];
    snprintf(names[ks - 2], 64, "splitK%d 1023x%dx1025 (batch)", ks, (int)p.K);
    shapes.push_back({names[ks - 2], p});
  }
  for (auto& s : shapes) {
    const double flops = 2.0 * s.p.M * s.p.N * s.p.K * s.p.batch;
    const size_t outn = s.p.M * s.p.N * s.p.batch;  // ldc == M here
    GemmProblem pr = s.p; pr.C = Cref;
    launch_gemm_cfg<C1>(pr, EpiStore{}, 0);
    auto report = [&](const char* cname, float ms) {
      cudaMemset(d, 0, 8);
      maxdiff<<<512, 256>>>(C, Cref, outn, d);
      double md; cudaMemcpy(&md, d, 8, cudaMemcpyDeviceToHost);
      printf("%-36s %-24s %8.3f ms %6.2f TFLOP/s  maxdiff %.1e\n", s.name, cname, ms, flops / ms / 1e9, md);
    };
    const int reps = s.p.N > 10000 || s.p.batch > 1 ? 3 : 20;
    report("C1 128x128x16 s4 8w", run<C1>(s.p, reps));
    report("C9 128x64x16 s3 x2", run<C9>(s.p, reps));
    report("C10 128x64x32 s2 x2", run<C10>(s.p, reps));
    report("C11 128x64x16 s4 x2", run<C11>(s.p, reps));
    report("C5 64x64x16 s4 x3", run<C5>(s.p, reps));
    report("C12 64x64x16 s3 x3", run<C12>(s.p, reps));
    report("C13 64x128x16 s3 x2", run<C13>(s.p, reps));
    report("C14 64x64x32 s2 x3", run<C14>(s.p, reps));
    report("C15 32x64x32 s2 x4 2w", run<C15>(s.p, reps));
    report("C16 64x32x32 s2 x4 2w", run<C16>(s.p, reps));
    report("C17 32x32x32 s2 x8 1w", run<C17>(s.p, reps));
    report("C18 64x64x16 s3 x3", run<C18>(s.p, reps));
    report("C19 64x64x32 s2 8w 32x16", run<C19>(s.p, reps));
    report("C20 64x64x32 s2 8w 16x32", run<C20>(s.p, reps));
    report("C21 64x64x32 s3 8w 32x16", run<C21>(s.p, reps));
    report("C22 48x64x48 s2 6w", run<C22>(s.p, reps));
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
