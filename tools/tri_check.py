"""Dev check of the line-solve axis-0 pass (heat_tridiag.cuh, STKG_TRIDIAG=1) against the
transform-based fused pass (STKG_TRIDIAG=0): device solves, 2-slice host chunks (carried
state), 2D/3D; then event-timed cfg3 / cfg5 solves of both.

    python tools/tri_check.py [--no-time]
"""
import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = str(Path(__file__).resolve().parent.parent)
SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1912_10082_b200 as stk
out = {}
for ndim, n, nt in [(2, 1023, 5), (2, 511, 4), (2, 255, 7), (2, 127, 6), (2, 63, 5), (3, 127, 4),
                    (3, 63, 3)]:
    rng = np.random.default_rng(7 * n + nt)
    F = rng.standard_normal((nt, n ** ndim))
    T = nt / (n + 1.0)
    p = stk.HeatPlan.p1_uniform(ndim, n, nt, T=T, transform="dst")
    Fd = torch.from_numpy(F).cuda()
    U = p.solve(Fd)
    out[f"u{ndim}_{n}"] = U.cpu().numpy()
    out[f"r{ndim}_{n}"] = np.array(p.residual(U, Fd)[0])
    pc = stk.HeatPlan.p1_uniform(ndim, n, nt, T=T, transform="dst", time_chunk=2)
    out[f"h{ndim}_{n}"] = pc.solve_host(F)
np.savez(sys.argv[2], **out)
"""


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


res = {}
with tempfile.TemporaryDirectory() as td:
    for v in ("1", "0"):
        f = os.path.join(td, f"t{v}.npz")
        subprocess.run([sys.executable, "-c", SCRIPT, ROOT, f], check=True,
                       env=dict(os.environ, STKG_TRIDIAG=v, STKG_FUSED="1"))
        res[v] = dict(np.load(f))
for k in sorted(res["1"]):
    a, b = res["1"][k], res["0"][k]
    if k[0] == "r":
        print(k, "relres tri", float(a), "dst", float(b))
    else:
        print(k, "tri vs dst", rel(a, b))
if "--no-time" not in sys.argv:
    for cfg in ("cfg3", "cfg5"):
        for env in ({"STKG_TRIDIAG": "1"}, {"STKG_TRIDIAG": "1", "STKG_OVERLAP": "0"},
                    {"STKG_TRIDIAG": "0"}):
            r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "solve_time.py"),
                                "--cfg", cfg], env=dict(os.environ, **env), capture_output=True,
                               text=True)
            print(cfg, env, r.stdout.strip()[-600:] or r.stderr[-600:])
