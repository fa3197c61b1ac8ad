"""Full-size parity at the BASELINE configurations (VERDICT r1 "full-size parity the driver can
verify"): every time slice of the headline cfg3 solve against the streamed numpy oracle and a
crank_nicolson prefix; config 4's refined wave solve against an independent extended-precision
residual; the refined solve's forward error against the oracle's refined direct solve."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def cfg3_solution(stk, cuda):
    """The headline device solve of cfg3 (default backend: half-length DST passes along the
    contiguous axis + the time-marching line-solve pass along axis 0), U copied to the host,
    and the GPU residual."""
    import torch
    from paper_1912_10082_b200 import inputs
    cfg = inputs.CONFIGS["cfg3"]
    plan = stk.HeatPlan.p1_uniform(cfg.ndim, cfg.n, cfg.nt, transform="dst")
    F = inputs.heat_rhs_device(cfg)
    U = plan.solve(F)
    relres, _ = plan.residual(U, F)
    assert plan.schedule() == "line_solve"
    # a second solve is bit-identical (no atomics / order dependence anywhere on the path)
    U2 = plan.solve(F)
    assert bool(torch.equal(U, U2))
    del U2
    Uh = U.cpu().numpy()
    del U, F, plan
    torch.cuda.empty_cache()
    return cfg, Uh, relres


def test_cfg3_every_slice_vs_streamed_oracle(orc, cfg3_solution):
    """cfg3 (2D 1023^2 x 1024, full-rank U[-1,1] F): all 1024 time slices of the GPU U against
    the numpy tensor-form solve_projected_heat_with (stk/sylvester.hpp:117-142) on scipy eigh
    eigenbases, streamed in 32-slice chunks with the recurrence carried (F regenerated on the
    host bit-identically).  North_star bar: ||U - U_ref||_F / ||U_ref||_F <= 1e-10 and the
    GPU residual ||F - B(U)|| / ||F|| <= 1e-10."""
    from paper_1912_10082_b200 import inputs
    cfg, U, relres = cfg3_solution
    assert relres <= 1e-10
    m, a = orc.fem1d_matrices(0.0, 1.0, cfg.n)
    d, c = orc.heat_time_matrices(cfg.nt)
    lam, X = orc.p1_pencil_eig(m, a)
    stream = orc.DecoupledStream([(lam, X)] * cfg.ndim, d, c)
    num = den = worst = 0.0
    t0 = time.perf_counter()
    for l0 in range(0, cfg.nt, 32):
        k = min(32, cfg.nt - l0)
        Fh = inputs.uniform_pm1(k * cfg.nx, 0, cfg.cid * 16, offset=l0 * cfg.nx).reshape(k, cfg.nx)
        Uref = stream.step(Fh)
        diff = U[l0:l0 + k] - Uref
        num += float(np.sum(diff * diff))
        den += float(np.sum(Uref * Uref))
        worst = max(worst, rel(U[l0:l0 + k], Uref))
    err = (num / den) ** 0.5
    print(f"cfg3 full: rel err {err:.3e} (worst chunk {worst:.3e}), relres {relres:.3e}, "
          f"oracle {time.perf_counter() - t0:.1f} s")
    assert err <= 1e-10 and worst <= 1e-10


def test_cfg3_prefix_vs_crank_nicolson(orc, cfg3_solution):
    """The first 128 slices of the cfg3 solve against the reference's own CPU method,
    crank_nicolson (stk/cn_baseline.hpp:26-48: factor M + dt/2 A once, march), with SuperLU in
    place of SimplicialLLT -- an algebra independent of the eigenbasis (the first k columns of
    U depend only on the first k columns of F)."""
    from paper_1912_10082_b200 import inputs
    cfg, U, _ = cfg3_solution
    k = 128
    m, a = orc.fem1d_matrices(0.0, 1.0, cfg.n)
    Fh = inputs.uniform_pm1(k * cfg.nx, 0, cfg.cid * 16).reshape(k, cfg.nx)
    t0 = time.perf_counter()
    Ucn = orc.crank_nicolson_splu([m] * 2, [a] * 2, 1.0 / cfg.nt, Fh)
    err = rel(U[:k], Ucn)
    print(f"cfg3 {k}-slice CN prefix: rel err {err:.3e} ({time.perf_counter() - t0:.1f} s)")
    assert err <= 1e-10


def _cfg4(stk):
    from paper_1912_10082_b200 import inputs
    cfg = inputs.CONFIGS["cfg4"]
    sm = stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, cfg.nh))
    tm = stk.wave_time_matrices(stk.TimeGrid(cfg.nt, 1.0))
    sb = np.stack([sm.M.band, sm.A.band, sm.Q.band])
    tb = np.stack([tm.Q.band, tm.D.band, tm.M.band])
    return cfg, sm, tm, sb, tb


def test_cfg4_refined_residual_extended_precision(stk, orc, cuda):
    """Config 4 (1D wave, cubic splines, 1023 x 1025): the refined solve's double-double
    residual (stkg_wave_residual_dd, stk/outer_krylov.hpp:159 true-residual semantics,
    WaveOperator::apply :178-186) checked independently at full size:
    (a) 2000 sampled entries of the residual vector against exact rational evaluation
        (Python Fractions) -- equal to FP64 rounding;
    (b) the relative residual against a 64-bit-mantissa band-by-band evaluation, within that
        evaluation's rounding floor; both below the north_star 1e-10 bar."""
    import torch
    from paper_1912_10082_b200 import inputs
    cfg, sm, tm, sb, tb = _cfg4(stk)
    plan = stk.WavePlan(sm, tm)
    b = inputs.wave_rhs_host(cfg).ravel()
    bd = torch.from_numpy(b).cuda()
    xh, xl, rep = plan.solve_refined(bd, tol=1e-10, inner_tol=1e-6, max_refine=6)
    assert rep.converged
    r_gpu = torch.empty_like(bd)
    rel_dd = plan.residual_dd(bd, xh, xl, out=r_gpu)
    xh_, xl_, r_gpu = xh.cpu().numpy(), xl.cpu().numpy(), r_gpu.cpu().numpy()
    idx = np.random.default_rng(5).choice(b.size, 2000, replace=False)
    for g, (r_ex, mag) in zip(idx, orc.wave_residual_exact_entries(sb, tb, b, xh_, xl_, idx)):
        assert abs(r_gpu[g] - r_ex) <= 4e-16 * abs(r_ex) + 1e-28 * mag, (g, r_gpu[g], r_ex)
    r = orc.wave_residual_banded(sb, tb, b, xh_, xl_)
    rel_ld = float(np.sqrt(np.sum(r * r)) / np.linalg.norm(b))
    floor = orc.wave_residual_floor(sb, tb, b, xh_, xl_)
    print(f"cfg4 refined: dd {rel_dd:.3e}  longdouble {rel_ld:.3e} (floor {floor:.1e})  "
          f"PCG its {rep.iterations}")
    assert rel_dd <= 1e-10 and rel_ld <= 1e-10
    assert abs(rel_dd - rel_ld) <= 4 * floor + 1e-3 * rel_dd


@pytest.mark.parametrize("nh,nt", [(127, 128), (255, 256)])
def test_wave_refined_forward_error_vs_oracle(stk, orc, cuda, nh, nt):
    """Forward error of the GPU refined wave solve against the oracle's refined direct solve
    (kron_direct_solve, stk/bench.hpp:414-429, SuperLU + longdouble iterative refinement):
    ||x - x_ref|| / ||x_ref|| <= 1e-10 (north_star bar); the FP64 direct solve alone is off by
    ~cond(B) eps (reported)."""
    import torch
    sm = stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, nh))
    tm = stk.wave_time_matrices(stk.TimeGrid(nt, 1.0))
    sb = np.stack([sm.M.band, sm.A.band, sm.Q.band])
    tb = np.stack([tm.Q.band, tm.D.band, tm.M.band])
    plan = stk.WavePlan(sm, tm)
    b = np.random.default_rng(nh).standard_normal(plan.N)
    xh, xl, rep = plan.solve_refined(torch.from_numpy(b).cuda(), tol=1e-13, inner_tol=1e-6)
    assert rep.converged
    x = xh.cpu().numpy().astype(np.longdouble) + xl.cpu().numpy().astype(np.longdouble)
    rh, rl, hist = orc.wave_refined_direct(sb, tb, b, steps=3)
    xr = rh.astype(np.longdouble) + rl.astype(np.longdouble)
    err = float(np.sqrt(np.sum((x - xr) ** 2) / np.sum(xr * xr)))
    print(f"wave {nh}x{nt + 1}: forward error {err:.3e}; oracle residual history {hist}")
    assert hist[-1] <= 1e-13
    assert err <= 1e-10


@pytest.mark.parametrize("nh,nt", [(63, 64), (127, 128)])
def test_wave_gmres_and_pcg_vs_oracle_mid_size(stk, orc, cuda, nh, nt):
    """GMRES (stk/outer_krylov.hpp:75-164) and PCG at mid sizes (the n <= 33 cases are in
    test_wave_gpu.py): iterates within their tolerance's forward-error envelope of the oracle
    refined direct solve; GMRES iteration count within 2 of the reference-faithful numpy
    GMRES (MGS + one re-orthogonalisation, Givens)."""
    import torch
    sm = stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, nh))
    tm = stk.wave_time_matrices(stk.TimeGrid(nt, 1.0))
    sb = np.stack([sm.M.band, sm.A.band, sm.Q.band])
    tb = np.stack([tm.Q.band, tm.D.band, tm.M.band])
    plan = stk.WavePlan(sm, tm)
    b = np.random.default_rng(nt).standard_normal(plan.N)
    rh, rl, _ = orc.wave_refined_direct(sb, tb, b, steps=2)
    xg, rep = plan.gmres(torch.from_numpy(b).cuda(), stk.GmresConfig(tol=1e-8, maxit=2000))
    xp, prep = plan.pcg(torch.from_numpy(b).cuda(), tol=1e-8, maxit=4000)
    assert rep.converged and prep.converged
    W = orc.WaveSystemNP(sb, tb)
    xo, its_o, hist_o = W.gmres(b, tol=1e-8, maxit=2000)
    print(f"wave {nh}: gmres its {rep.iterations} (oracle {its_o}), pcg its {prep.iterations}, "
          f"fwd err gmres {rel(xg.cpu().numpy().ravel(), rh):.2e} pcg {rel(xp.cpu().numpy().ravel(), rh):.2e}")
    assert abs(rep.iterations - its_o) <= 2
    assert rel(xg.cpu().numpy().ravel(), rh) <= 1e-5 and rel(xp.cpu().numpy().ravel(), rh) <= 1e-5
