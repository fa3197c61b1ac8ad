"""Debug: device solves of a 2D n = 1023 plan under STKG_OVERLAP=K (set in the environment),
compared with the numpy oracle's decoupled solve; prints per-slice relative errors."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch
import paper_1912_10082_b200 as stk
from oracle import oracle as O

n, nt = int(sys.argv[1]), int(sys.argv[2])
F = np.random.default_rng(n + nt).standard_normal((nt, n * n))
p = stk.HeatPlan.p1_uniform(2, n, nt, transform="dst")
Fd = torch.from_numpy(F).cuda()
U1 = p.solve(Fd).cpu().numpy()
U2 = p.solve(Fd).cpu().numpy()
m, a = O.fem1d_matrices(0.0, 1.0, n)
d, c = O.heat_time_matrices(nt)
lam, X = O.p1_pencil_eig(m, a)
Ur = O.heat_decoupled([(lam, X)] * 2, d, c, F)
e1 = np.linalg.norm(U1 - Ur, axis=1) / np.linalg.norm(Ur, axis=1)
e2 = np.linalg.norm(U2 - Ur, axis=1) / np.linalg.norm(Ur, axis=1)
print("run1", " ".join(f"{x:.1e}" for x in e1))
print("run2", " ".join(f"{x:.1e}" for x in e2))
print("repeat identical", np.array_equal(U1, U2))
