"""Full-size parity of the GPU heat solve against the numpy oracle ("compute
full U_ref once per seed, in streaming fashion, column by column").

The device solves the whole configuration (F generated in place by the counter generator);
the oracle then marches over the time slices in chunks -- F regenerated on the host
bit-identically, transformed with scipy eigh eigenbases (independent of the product's
closed form), the modal recurrence carried across chunks, transformed back -- and each
chunk of U is compared with the GPU's.  Writes a JSON summary.

    python tools/full_parity.py [cfg3|cfg2|cfg5] [--transform dst|dense] [--out FILE]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_10082_b200 as stk  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1912_10082_b200 import inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="cfg3")
ap.add_argument("--transform", default="dst")
ap.add_argument("--chunk", type=int, default=32)
ap.add_argument("--out", default=None)
ap.add_argument("--oracle", choices=["decoupled", "cn"], default="decoupled",
                help="cn: the reference's crank_nicolson (SuperLU), an independent algebra")
a = ap.parse_args()
cfg = inputs.CONFIGS[a.config]
nx, nt, nd = cfg.nx, cfg.nt, cfg.ndim

plan = stk.HeatPlan.p1_uniform(nd, cfg.n, nt, transform=a.transform)
F = inputs.heat_rhs_device(cfg)
t0 = time.perf_counter()
U = plan.solve(F)
torch.cuda.synchronize()
t_gpu = time.perf_counter() - t0
relres, _ = plan.residual(U, F)
del F
torch.cuda.empty_cache()

m, aa = O.fem1d_matrices(0.0, 1.0, cfg.n)
d, c = O.heat_time_matrices(nt)
lam, X = O.p1_pencil_eig(m, aa)
ns = [cfg.n] * nd
lam_t = np.zeros(ns)
for ax in range(nd):
    shape = [1] * nd
    shape[ax] = cfg.n
    lam_t = lam_t + lam.reshape(shape)
if cfg.rank > 0:
    left, right = inputs.heat_factors(cfg)
y = np.zeros(ns)
num = den = 0.0
worst = 0.0
t0 = time.perf_counter()
if a.oracle == "cn":
    import scipy.sparse.linalg as spl
    Msp, Asp = O.tensor_sparse([m] * nd, [aa] * nd)
    dt = 1.0 / nt
    lu = spl.splu((Msp + (dt / 2.0) * Asp).tocsc())
    rhs_op = (Msp - (dt / 2.0) * Asp).tocsr()
    u = np.zeros(nx)
for l0 in range(0, nt, a.chunk):
    k = min(a.chunk, nt - l0)
    if cfg.rank == 0:
        Fh = inputs.uniform_pm1(k * nx, 0, cfg.cid * 16, offset=l0 * nx).reshape(k, *ns)
    else:
        Fh = (right[l0:l0 + k] @ left.T).reshape(k, *ns)
    if a.oracle == "cn":  # (M + dt/2 A) u_l = (M - dt/2 A) u_{l-1} + F_l (stk/cn_baseline.hpp)
        Uref = np.empty((k, nx))
        Fk = Fh.reshape(k, nx)
        for j in range(k):
            u = lu.solve(rhs_op @ u + Fk[j])
            Uref[j] = u
    else:
        G = Fh
        for ax in range(nd):
            G = np.moveaxis(np.tensordot(G, X, axes=([ax + 1], [0])), -1, ax + 1)
        Y = np.empty_like(G)
        for j in range(k):
            lj = l0 + j
            rhs = G[j]
            if lj > 0:
                rhs = rhs - (d[1][lj - 1] + lam_t * c[1][lj - 1]) * y
            y = rhs / (d[0][lj] + lam_t * c[0][lj])
            Y[j] = y
        for ax in range(nd):
            Y = np.moveaxis(np.tensordot(Y, X, axes=([ax + 1], [1])), -1, ax + 1)
        Uref = Y.reshape(k, nx)
    Ug = U[l0:l0 + k].cpu().numpy()
    diff = Ug - Uref
    num += float(np.sum(diff * diff))
    den += float(np.sum(Uref * Uref))
    worst = max(worst, float(np.linalg.norm(diff) / max(np.linalg.norm(Uref), 1e-300)))
t_cpu = time.perf_counter() - t0
res = {"config": cfg.name, "transform": a.transform, "slices_compared": nt,
       "rel_error_full": (num / den) ** 0.5, "worst_chunk_rel_error": worst,
       "gpu_relres_k1": relres, "gpu_solve_s": t_gpu, "oracle_stream_s": t_cpu,
       "oracle": ("crank_nicolson (stk/cn_baseline.hpp:26-48) with SuperLU, marched over all "
                  "slices" if a.oracle == "cn" else
                  "numpy tensor-form solve_projected_heat_with, scipy eigh eigenbases, "
                  f"streamed in chunks of {a.chunk} slices with the recurrence carried")}
print(json.dumps(res))
if a.out:
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
assert res["rel_error_full"] <= 1e-10 and relres <= 1e-10, res
