"""Time the K1 residual kernel (heat_apply_kernel<ndim, residual>) on cfg3 / cfg5 shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1912_10082_b200 as stk
from paper_1912_10082_b200 import inputs
for name, nt in (("cfg3", 1024), ("cfg5", 256), ("cfg1", 256)):
    cfg = inputs.CONFIGS[name]
    plan = stk.HeatPlan.p1_uniform(cfg.ndim, cfg.n, nt, transform="dst")
    F = torch.empty((nt, cfg.nx), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    U = plan.solve(F)
    for _ in range(2):
        plan.residual(U, F)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        rr, _ = plan.residual(U, F)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    N = cfg.nx * nt
    print(f"{name}: residual {ms:.3f} ms  {16 * N / ms / 1e6:.0f} GB/s  relres {rr:.2e}")
    del U, F, plan
    torch.cuda.empty_cache()
