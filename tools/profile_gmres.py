"""ncu driver: GMRES on config 4 for a given number of iterations (default 60)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1912_10082_b200 as stk  # noqa: E402
from paper_1912_10082_b200 import inputs  # noqa: E402

cfg = inputs.CONFIGS["cfg4"]
plan = stk.WavePlan(stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, cfg.nh)),
                    stk.wave_time_matrices(stk.TimeGrid(cfg.nt, 1.0)))
F = torch.from_numpy(inputs.wave_rhs_host(cfg)).cuda()
its = int(sys.argv[1]) if len(sys.argv) > 1 else 60
x, rep = plan.gmres(F, stk.GmresConfig(tol=1e-12, maxit=its))
torch.cuda.synchronize()
print("gmres", rep.iterations, rep.final_relres, rep.wall_time_s)
