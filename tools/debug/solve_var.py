"""Run-to-run spread of the cfg3 device solve: 30 individually event-timed solves, then 5
batches of 5 back-to-back solves, then 5 profiled solves (per-class kernel times)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import torch
import paper_1912_10082_b200 as stk
from paper_1912_10082_b200 import inputs
cfg = inputs.CONFIGS["cfg3"]
plan = stk.HeatPlan.p1_uniform(cfg.ndim, cfg.n, cfg.nt, transform="dst")
F = inputs.heat_rhs_device(cfg)
U = torch.empty_like(F)
for _ in range(3):
    plan.solve(F, out=U)
torch.cuda.synchronize()
def timed(k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        plan.solve(F, out=U)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k
print("single", " ".join(f"{timed(1):.2f}" for _ in range(30)))
print("batch5", " ".join(f"{timed(5):.2f}" for _ in range(5)))
for _ in range(5):
    plan.profile_begin()
    plan.solve(F, out=U)
    torch.cuda.synchronize()
    print("prof", plan.profile_end())
