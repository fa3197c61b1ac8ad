"""Event-timed K1 residual on the cfg5 geometry (3D 127^3), n_t slices (default 256)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import paper_1912_10082_b200 as stk  # noqa: E402

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n = 127
plan = stk.HeatPlan.p1_uniform(3, n, nt, transform="dst")
U = torch.empty((nt, n ** 3), dtype=torch.float64, device="cuda").uniform_(-1, 1)
F = torch.empty_like(U).uniform_(-1, 1)
for _ in range(2):
    plan.residual(U, F)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    r = plan.residual(U, F)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
N = n ** 3 * nt
print(f"3D K1 residual nt={nt}: {ms:.3f} ms, {16 * N / ms / 1e6:.0f} GB/s, relres {r[0]:.3e}")
