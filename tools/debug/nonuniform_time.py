"""cfg3-size solve on a NON-uniform time grid (random step sizes around cfg3's dt): the
line-solve pass with per-step constants vs the fused transform pass (STKG_TRI_NONUNIFORM=0)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import numpy as np
import torch
import paper_1912_10082_b200 as stk
from paper_1912_10082_b200 import inputs
cfg = inputs.CONFIGS["cfg3"]
n, nt = cfg.n, cfg.nt
rng = np.random.default_rng(1)
dt = rng.uniform(0.5, 1.5, nt) / nt
g = stk.SpaceGrid1D(0.0, 1.0, n)
e = stk.p1_eigpair(g)
M, A = stk.fem1d_matrices(g)
D = stk.Bidiagonal(np.ones(nt), -np.ones(nt - 1))
Cm = stk.Bidiagonal(0.5 * dt, 0.5 * dt[1:])
plan = stk.HeatPlan(stk.TensorEigPair([e, e]), D, Cm, [M, M], [A, A], transform="dst",
                    p1_h=[g.fem_h] * 2)
F = inputs.heat_rhs_device(cfg)
U = torch.empty_like(F)
for _ in range(2):
    plan.solve(F, out=U)
torch.cuda.synchronize()
ms = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); plan.solve(F, out=U); e1.record(); torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
plan.profile_begin(); plan.solve(F, out=U); torch.cuda.synchronize()
print(plan.schedule(), "ms", min(ms), plan.profile_end(), "relres", plan.residual(U, F)[0])
