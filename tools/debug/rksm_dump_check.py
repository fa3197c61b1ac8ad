"""Debug aid: run one 2D RKSM solve with STKG_RKSM_DUMP and check the dumped state."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from oracle import oracle as orc
import paper_1912_10082_b200 as stk

out = "gpurun_out/rksm_dump"
os.makedirs(out, exist_ok=True)
os.environ["STKG_RKSM_DUMP"] = out
n, nt, iters = 31, 20, int(sys.argv[2]) if len(sys.argv) > 2 else 6
transform = sys.argv[1] if len(sys.argv) > 1 else "dense"
h = 1.0 / (n + 1)
f = np.cos(np.pi / 2 * np.arange(1, n + 1) * h) * h
rng = np.random.default_rng(5)
L = np.vstack([np.kron(f, f)[None], rng.standard_normal((1, n * n))])
tt = (np.arange(nt) + 0.5) / nt
R = np.vstack([(10 * np.sin(tt) * tt / nt)[None], rng.standard_normal((1, nt))])
plan = stk.HeatPlan.p1_uniform(2, n, nt, transform=transform)
dev = lambda a: torch.tensor(a, dtype=torch.float64, device="cuda")
UL, UR, rep = plan.rksm(dev(L), dev(R), fixed_iters=iters)
print("hist", rep.rel_res_history)
rd = lambda name: np.fromfile(f"{out}/{name}.bin")
nx, kv, km, q, k, rf = [int(x) for x in rd("dims")]
V = rd("V").reshape(kv, nx).T
MV = rd("MV").reshape(km, nx).T
AV = rd("AV").reshape(km, nx).T
Q = rd("Q").reshape(q, nx).T
T = rd("T").reshape(-1, q).T
y = rd("y").reshape(nt, k).T
m, a = orc.fem1d_matrices(0.0, 1.0, n)
d, c = orc.heat_time_matrices(nt)
M, A = orc.tensor_sparse([m, m], [a, a])
print("dims", nx, kv, km, q, k, rf)
print("VtV-I", np.abs(V.T @ V - np.eye(kv)).max())
print("QtQ-I", np.abs(Q.T @ Q - np.eye(q)).max())
print("MV err", np.abs(MV - M @ V[:, :km]).max() / np.abs(MV).max())
print("AV err", np.abs(AV - A @ V[:, :km]).max() / np.abs(AV).max())
f1 = V[:, :rf]
Tx = Q.T @ np.hstack([f1, MV, AV])
print("T err", np.abs(T - Tx).max() / np.abs(Tx).max())
Vk = V[:, :k]
P = np.hstack([f1, MV, AV])
print("span resid of [f1 MV AV] outside Q", np.linalg.norm(P - Q @ (Q.T @ P)) / np.linalg.norm(P))
Dm, Cm = orc.bidiag_dense(d), orc.bidiag_dense(c)
F = L.T @ R
Rfull = M @ Vk @ y @ Dm + A @ Vk @ y @ Cm - F
print("true relres of V y", np.linalg.norm(Rfull) / np.linalg.norm(F))
# Galerkin check
print("Galerkin Vt R", np.linalg.norm(Vk.T @ Rfull) / np.linalg.norm(F))
# shifted-solve check: each new block should lie in span of (A - s M)^-1 M V_prev
