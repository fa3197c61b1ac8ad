"""STKG_DST_BULK=1 (bulk-copy input of the contiguous DST pass) against the default: same
solve bit for bit (the arithmetic is unchanged), then timing of both."""
import os, subprocess, sys, tempfile
from pathlib import Path
import numpy as np
ROOT = str(Path(__file__).resolve().parent.parent.parent)
SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1912_10082_b200 as stk
out = {}
for n, nt in [(1023, 5), (1023, 4)]:
    F = np.random.default_rng(n + nt).standard_normal((nt, n * n))
    p = stk.HeatPlan.p1_uniform(2, n, nt, T=nt / 1024.0, transform="dst")
    out[f"u{nt}"] = p.solve(torch.from_numpy(F).cuda()).cpu().numpy()
np.savez(sys.argv[2], **out)
"""
res = {}
with tempfile.TemporaryDirectory() as td:
    for v in ("1", "0"):
        f = os.path.join(td, f"b{v}.npz")
        subprocess.run([sys.executable, "-c", SCRIPT, ROOT, f], check=True,
                       env=dict(os.environ, STKG_DST_BULK=v))
        res[v] = dict(np.load(f))
for k in res["1"]:
    print(k, "bit-identical" if np.array_equal(res["1"][k], res["0"][k]) else
          float(np.abs(res["1"][k] - res["0"][k]).max()))
for r in range(2):
    for v in ("0", "1"):
        o = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "solve_time.py"), "--cfg", "cfg3",
                            "--reps", "3"], env=dict(os.environ, STKG_DST_BULK=v),
                           capture_output=True, text=True).stdout
        print("BULK=" + v, o.strip()[:260])
