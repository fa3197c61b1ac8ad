"""PCIe bound of the end-to-end heat solve: pinned H2D / D2H bandwidth alone and together,
and the e2e solve (stkg_heat_solve_host) at several pipeline chunk sizes (cfg3)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1912_10082_b200 as stk
from paper_1912_10082_b200 import inputs

GB = 2 << 30
h_a = torch.empty(GB // 8, dtype=torch.float64).pin_memory()
h_b = torch.empty(GB // 8, dtype=torch.float64).pin_memory()
d_a = torch.empty(GB // 8, dtype=torch.float64, device="cuda")
d_b = torch.empty(GB // 8, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def bw(h2d, d2h):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(3):
        if h2d:
            with torch.cuda.stream(s1): d_a.copy_(h_a, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h_b.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    return 3 * GB / dt / 1e9
print("H2D alone GB/s %.1f" % bw(True, False))
print("D2H alone GB/s %.1f" % bw(False, True))
print("both (each) GB/s %.1f" % bw(True, True))
del h_a, h_b, d_a, d_b
torch.cuda.empty_cache()
cfg = inputs.CONFIGS["cfg3"]
N = cfg.unknowns
Fh = torch.empty((cfg.nt, cfg.nx), dtype=torch.float64).pin_memory()
Uh = torch.empty_like(Fh).pin_memory()
Fh.copy_(inputs.heat_rhs_device(cfg).cpu())
for tc in [int(x) for x in (sys.argv[1:] or ["8", "16", "32", "64", "128"])]:
    plan = stk.HeatPlan.p1_uniform(2, cfg.n, cfg.nt, transform="dst", time_chunk=tc)
    plan.solve_host(Fh.numpy(), out=Uh.numpy())
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(2):
        plan.solve_host(Fh.numpy(), out=Uh.numpy())
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 2
    print("time_chunk %4d slices (%5.0f MB): %.3f s  e2e %.3e unk/s  (%.1f GB/s each way)"
          % (tc, tc * cfg.nx * 8 / 2**20, dt, N / dt, N * 8 / dt / 1e9))
    plan.close()
