"""Does splitting H2D / D2H over several streams (copy engines) raise the concurrent
bidirectional pinned bandwidth?"""
import time
import torch

GB = 2 << 30
n = GB // 8
h_a = torch.empty(n, dtype=torch.float64).pin_memory()
h_b = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
for k in (1, 2, 4):
    s_up = [torch.cuda.Stream() for _ in range(k)]
    s_dn = [torch.cuda.Stream() for _ in range(k)]
    part = n // k
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        for i in range(k):
            sl = slice(i * part, (i + 1) * part)
            with torch.cuda.stream(s_up[i]):
                d_a[sl].copy_(h_a[sl], non_blocking=True)
            with torch.cuda.stream(s_dn[i]):
                h_b[sl].copy_(d_b[sl], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{k} stream(s) per direction: {3 * GB / dt / 1e9:.1f} GB/s each way (concurrent)")
