"""Small-size runs of every heat and wave device path (a quick smoke; also the driver for
compute-sanitizer where a pool allows it -- this one does not):
    python tools/sanitize.py
Covers the padded-layout DST passes (contiguous, 16-byte strided in place, lane-segment
FFTs), the unpadded strided kernel, the chunked and one-chain scans, the factored scan, the
x-marching K1 kernels (2D/3D, chunked time grid) and the generic 1D one, the host-buffer
pipeline, the DMMA backend, and the wave operator / preconditioner / PCG."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_10082_b200 as stk  # noqa: E402

rng = np.random.default_rng(0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


for ndim, n, nt in [(2, 127, 5), (2, 63, 70), (3, 31, 4), (2, 1023, 2), (3, 15, 3), (1, 63, 9)]:
    for tr in ("dst", "dense"):
        p = stk.HeatPlan.p1_uniform(ndim, n, nt, transform=tr, time_chunk=3)
        F = rng.standard_normal((nt, n ** ndim))
        U = p.solve(dev(F))
        rr, _ = p.residual(U, dev(F))
        Uh = p.solve_host(F)
        L, R = rng.standard_normal((2, n ** ndim)), rng.standard_normal((2, nt))
        p.solve_factored(dev(L), dev(R))
        p.apply(U)
        print(ndim, n, nt, tr, "relres", rr, flush=True)

# the line-solve schedule (mesh-proportional time steps; 2D full wave of tiles, 2D / 3D
# latency-bound tile counts, carried chunks, a non-uniform time grid)
for ndim, n, nt in [(2, 1023, 5), (2, 511, 4), (3, 127, 3)]:
    p = stk.HeatPlan.p1_uniform(ndim, n, nt, T=nt / (n + 1.0), transform="dst", time_chunk=2)
    F = rng.standard_normal((nt, n ** ndim))
    U = p.solve(dev(F))
    rr, _ = p.residual(U, dev(F))
    p.solve_host(F)
    print(ndim, n, nt, p.schedule(), "relres", rr, flush=True)
    assert p.schedule() == "line_solve"
g = stk.SpaceGrid1D(0.0, 1.0, 511)
e = stk.p1_eigpair(g)
M, A = stk.fem1d_matrices(g)
D = stk.Bidiagonal(rng.uniform(1.0, 2.0, 4), rng.uniform(-1.0, -0.2, 3))
Cm = stk.Bidiagonal(rng.uniform(1e-3, 2e-3, 4), rng.uniform(1e-3, 2e-3, 3))
pn = stk.HeatPlan(stk.TensorEigPair([e, e]), D, Cm, [M, M], [A, A], transform="dst",
                  p1_h=[g.fem_h] * 2)
F = rng.standard_normal((4, 511 * 511))
print("non-uniform", pn.schedule(), "relres", pn.residual(pn.solve(dev(F)), dev(F))[0], flush=True)

sm = stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, 31))
tm = stk.wave_time_matrices(stk.TimeGrid(32, 1.0))
wp = stk.WavePlan(sm, tm)
b = dev(rng.standard_normal((tm.M.n, sm.M.n)))
wp.apply(b)
x, rep = wp.pcg(b, tol=1e-8, maxit=50)
print("wave pcg", rep.iterations, rep.final_relres)
torch.cuda.synchronize()
print("sanitize run ok")
