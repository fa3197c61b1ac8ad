"""Debug: the overlap test's sequence of plans in one process, each solve checked against the
numpy oracle per slice (STKG_OVERLAP from the environment)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch
import paper_1912_10082_b200 as stk
from oracle import oracle as O

for n, nt in [(1023, 40), (1023, 37), (511, 64)]:
    F = np.random.default_rng(n + nt).standard_normal((nt, n * n))
    p = stk.HeatPlan.p1_uniform(2, n, nt, transform="dst")
    Fd = torch.from_numpy(F).cuda()
    U = p.solve(Fd)
    U1 = U.cpu().numpy()
    U2 = p.solve(Fd).cpu().numpy()
    rr = p.residual(U, Fd)[0]
    m, a = O.fem1d_matrices(0.0, 1.0, n)
    d, c = O.heat_time_matrices(nt)
    lam, X = O.p1_pencil_eig(m, a)
    Ur = O.heat_decoupled([(lam, X)] * 2, d, c, F)
    e1 = np.linalg.norm(U1 - Ur, axis=1) / np.linalg.norm(Ur, axis=1)
    e2 = np.linalg.norm(U2 - Ur, axis=1) / np.linalg.norm(Ur, axis=1)
    print(n, nt, "max err run1 %.2e at %d, run2 %.2e at %d, relres %.2e, repeat identical %s" % (
        e1.max(), e1.argmax(), e2.max(), e2.argmax(), rr, np.array_equal(U1, U2)))
