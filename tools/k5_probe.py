"""Time the wave operator (K5) and one PCG iteration on config 4."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1912_10082_b200 as stk
from paper_1912_10082_b200 import inputs
cfg = inputs.CONFIGS["cfg4"]
plan = stk.WavePlan(stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, cfg.nh)),
                    stk.wave_time_matrices(stk.TimeGrid(cfg.nt, 1.0)))
x = torch.randn(plan.N, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(5):
    plan.apply(x, y)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(100):
    plan.apply(x, y)
e1.record()
torch.cuda.synchronize()
us = 1e3 * e0.elapsed_time(e1) / 100
print(f"K5 apply {us:.1f} us  {16 * plan.N / us / 1e3:.0f} GB/s")
F = torch.from_numpy(inputs.wave_rhs_host(cfg)).cuda()
_, rep = plan.pcg(F, tol=1e-7, maxit=6000)
print(f"PCG {rep.iterations} its {rep.wall_time_s:.3f} s {1e3 * rep.wall_time_s / rep.iterations:.3f} ms/it")
