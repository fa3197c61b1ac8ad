"""Small driver for ncu captures of the heat solve kernels (same kernels as bench.py, fewer
time slices so that ncu's replay save/restore stays small)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1912_10082_b200 as stk  # noqa: E402
from paper_1912_10082_b200 import inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1023)
ap.add_argument("--ndim", type=int, default=2)
ap.add_argument("--nt", type=int, default=64)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--transform", default="dense")
a = ap.parse_args()
cfg = inputs.HeatConfig("profile", a.ndim, a.n, a.nt, 0, 3)
g = stk.SpaceGrid1D(0.0, 1.0, a.n)
M, A = stk.fem1d_matrices(g)
D, Cm = stk.heat_time_matrices(stk.TimeGrid(a.nt, 1.0))
plan = stk.HeatPlan.p1_uniform(a.ndim, a.n, a.nt, transform=a.transform)
F = inputs.heat_rhs_device(cfg)
U = torch.empty_like(F)
import time
for _ in range(a.reps):
    plan.solve(F, out=U)
torch.cuda.synchronize()
plan.profile_begin()
t0 = time.perf_counter()
plan.solve(F, out=U)
torch.cuda.synchronize()
print("solve ms", 1e3 * (time.perf_counter() - t0), plan.profile_end())
print("relres", plan.residual(U, F)[0])
