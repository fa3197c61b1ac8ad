"""cuBLAS FP64 GEMM reference point (torch.matmul float64) at the heat transform shapes."""
import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
d = torch.device("cuda:0")
for (m, k, n, b) in [(1023, 1023, 1023, 64), (1024, 1024, 1024, 64), (1023, 1023, 1023 * 256, 1), (4096, 4096, 4096, 1), (8192,8192,8192,1)]:
    A = torch.randn(b, m, k, dtype=torch.float64, device=d) if b > 1 else torch.randn(m, k, dtype=torch.float64, device=d)
    B = torch.randn(b, k, n, dtype=torch.float64, device=d) if b > 1 else torch.randn(k, n, dtype=torch.float64, device=d)
    for _ in range(3): C = A @ B
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 5
    for _ in range(reps): C = A @ B
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cuBLAS DGEMM m{m} k{k} n{n} batch{b}: {2.0*m*n*k*b/ms/1e9:.2f} TFLOP/s ({ms:.2f} ms)")
    del A, B, C
