"""Per-kernel-class split of a heat config's device solve (profiled, kernels back to back):
python tools/cfg_breakdown.py cfg5"""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import paper_1912_10082_b200 as stk  # noqa: E402
from paper_1912_10082_b200 import inputs  # noqa: E402

cfg = inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5"]
plan = stk.HeatPlan.p1_uniform(cfg.ndim, cfg.n, cfg.nt, transform="dst")
F = inputs.heat_rhs_device(cfg)
U = torch.empty_like(F)
for _ in range(3):
    plan.solve(F, out=U)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    plan.solve(F, out=U)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
plan.profile_begin()
plan.solve(F, out=U)
prof = plan.profile_end()
print(json.dumps({"cfg": cfg.name, "ms": ms, "profile": prof}))
