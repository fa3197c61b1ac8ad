"""RKSM on the BASELINE low-rank configs (cfg1/2/5): iterations, relres, wall time, unk/s,
next to the direct decoupled solve of the same factored load."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1912_10082_b200 as stk
from paper_1912_10082_b200 import inputs

for name in sys.argv[1:] or ["cfg1", "cfg2", "cfg5"]:
    cfg = inputs.CONFIGS[name]
    left, right = inputs.heat_factors(cfg)
    L = torch.tensor(left.T.copy(), device="cuda")
    R = torch.tensor(right.T.copy(), device="cuda")
    plan = stk.HeatPlan.p1_uniform(cfg.ndim, cfg.n, cfg.nt, transform="dst")
    for maxit in (100,):
        plan.rksm(L, R, maxit=3)  # warm
        torch.cuda.synchronize()
        t = time.perf_counter()
        UL, UR, rep = plan.rksm(L, R, maxit=maxit)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        plan.solve_factored(L, R)
        torch.cuda.synchronize()
        t = time.perf_counter()
        U = plan.solve_factored(L, R)
        torch.cuda.synchronize()
        dd = time.perf_counter() - t
        print(json.dumps({"cfg": name, "its": rep.iterations, "relres": rep.final_relres,
                          "converged": rep.converged, "rank": rep.rank, "rksm_s": dt,
                          "rksm_unk_s": cfg.nx * cfg.nt / dt, "direct_s": dd,
                          "direct_unk_s": cfg.nx * cfg.nt / dd,
                          "hist_tail": rep.rel_res_history[-3:]}))
