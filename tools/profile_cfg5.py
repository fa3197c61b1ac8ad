"""cfg5 (3D 127^3 x 256, rank-8 factored load): per-launch timing of the direct solve."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import paper_1912_10082_b200 as stk  # noqa: E402
from paper_1912_10082_b200 import inputs  # noqa: E402
cfg = inputs.CONFIGS["cfg5"]
left, right = inputs.heat_factors(cfg)
L = torch.tensor(left.T.copy(), device="cuda")
R = torch.tensor(right.T.copy(), device="cuda")
plan = stk.HeatPlan.p1_uniform(3, cfg.n, cfg.nt, transform="dst")
U = plan.solve_factored(L, R)
F = torch.empty_like(U)
for _ in range(3):
    plan.solve_factored(L, R)
torch.cuda.synchronize()
plan.profile_begin()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
plan.solve_factored(L, R)
e1.record()
torch.cuda.synchronize()
print("factored solve ms", e0.elapsed_time(e1), plan.profile_end())
Fd = torch.empty((cfg.nt, cfg.nx), dtype=torch.float64, device="cuda").uniform_(-1, 1)
for _ in range(2):
    plan.solve(Fd, out=U)
torch.cuda.synchronize()
plan.profile_begin()
e0.record()
plan.solve(Fd, out=U)
e1.record()
torch.cuda.synchronize()
print("dense-F solve ms", e0.elapsed_time(e1), plan.profile_end())
