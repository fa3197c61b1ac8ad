"""Event-timed device solves of the bench workloads (A/B helper for kernel variants selected by
environment switches, e.g. STKG_FUSED=0/1):

    python tools/solve_time.py --cfg cfg3 --reps 5
prints one JSON line: per-solve ms (mean / min), unknowns/s, GPU residual, kernel-class split.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1912_10082_b200 as stk  # noqa: E402
from paper_1912_10082_b200 import inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg3")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--nt", type=int, default=0, help="override n_t (0: the config's)")
ap.add_argument("--transform", default="dst")
a = ap.parse_args()
cfg = inputs.CONFIGS[a.cfg] if hasattr(inputs, "CONFIGS") else None
if cfg is None:
    raise SystemExit("inputs.CONFIGS missing")
if a.nt:
    cfg = inputs.HeatConfig(cfg.name, cfg.ndim, cfg.n, a.nt, cfg.rank, cfg.cid)
plan = stk.HeatPlan.p1_uniform(cfg.ndim, cfg.n, cfg.nt, transform=a.transform)
F = inputs.heat_rhs_device(cfg)
U = torch.empty_like(F)
for _ in range(2):
    plan.solve(F, out=U)
torch.cuda.synchronize()
ms = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.solve(F, out=U)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
plan.profile_begin()
plan.solve(F, out=U)
torch.cuda.synchronize()
prof = plan.profile_end()
rr = plan.residual(U, F)[0]
unk = cfg.ndim and cfg.n ** cfg.ndim * cfg.nt
print(json.dumps({"cfg": a.cfg, "nt": cfg.nt, "ms_mean": sum(ms) / len(ms), "ms_min": min(ms),
                  "unknowns_per_s": unk / (min(ms) * 1e-3), "relres": rr, "profile": prof}))
