"""GPU parity tests of the wave hot path: K5 WaveOperator::apply, K2 TwoTermPrecond::solve,
K4 GMRES orthogonalisation and the PCG path, against the oracle and the SPEC known answers."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def host(t):
    return t.cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def band_from_dense(Dm):
    n = Dm.shape[0]
    b = np.zeros((7, n))
    for d in range(7):
        for i in range(n):
            j = i + d - 3
            if 0 <= j < n:
                b[d, i] = Dm[i, j]
    return b


def plan_from_bands(stk, sb, tb, precond=True):
    sm = stk.WaveSpaceMatrices(*(stk.Band7(sb[k]) for k in range(3)))
    tm = stk.WaveTimeMatrices(*(stk.Band7(tb[k]) for k in range(3)))
    return stk.WavePlan(sm, tm, precond=precond)


def plan_from_dense(stk, Mh, Ah, Qh, Qt, Dt, Mt, precond=True):
    sb = np.stack([band_from_dense(x) for x in (Mh, Ah, Qh)])
    tb = np.stack([band_from_dense(x) for x in (Qt, Dt, Mt)])
    return plan_from_bands(stk, sb, tb, precond)


@pytest.mark.parametrize("key", [("16_3", "16_3"), ("8_2", "5_2"), ("31_3", "33_3"),
                                 ("1023_3", "1024_3")])
def test_wave_apply_vs_oracle(stk, orc, ref_bands, cuda, key):
    sb, tb = ref_bands[f"space_{key[0]}"], ref_bands[f"time_{key[1]}"]
    plan = plan_from_bands(stk, sb, tb, precond=False)
    rng = np.random.default_rng(4)
    U = rng.standard_normal((tb.shape[2], sb.shape[2]))
    y = host(plan.apply(dev(U)))
    assert rel(y, orc.wave_apply(sb, tb, U)) < 1e-13


def test_wave_apply_kats(stk, cuda):
    # M = Q = I, D = 0 -> x -> 2x ; SPEC.md:464 symmetry with symmetric factors
    n, m = 6, 5
    I6, I5 = np.eye(n), np.eye(m)
    plan = plan_from_dense(stk, I6, np.zeros((n, n)), I6, I5, np.zeros((m, m)), I5, precond=False)
    x = np.random.default_rng(0).standard_normal((m, n))
    assert np.allclose(host(plan.apply(dev(x))), 2 * x, rtol=0, atol=0)
    rng = np.random.default_rng(1)
    sym = [(lambda B: np.triu(np.tril(B + B.T, 3), -3))(rng.standard_normal((k, k)))
           for k in (n, n, n, m, m, m)]
    plan = plan_from_dense(stk, *sym, precond=False)
    x, y = rng.standard_normal((2, m, n))
    xy = np.vdot(x, host(plan.apply(dev(y))))
    yx = np.vdot(y, host(plan.apply(dev(x))))
    assert abs(xy - yx) <= 1e-12 * abs(xy)


def test_two_term_solve_kats(stk, cuda):
    # SPEC.md:325 all scalars 1, V=[2] -> W=[1];  SPEC.md:326 identities -> V/2
    one = np.eye(1)
    plan = plan_from_dense(stk, one, 0 * one, one, one, 0 * one, one)
    assert host(plan.two_term_solve(dev([[2.0]])))[0, 0] == 1.0
    plan = plan_from_dense(stk, np.eye(7), np.zeros((7, 7)), np.eye(7), np.eye(4), np.zeros((4, 4)),
                           np.eye(4))
    V = np.random.default_rng(2).standard_normal((4, 7))
    assert np.allclose(host(plan.two_term_solve(dev(V))), V / 2, rtol=1e-15, atol=1e-15)


def test_two_term_solve_random_pencils_and_round_trip(stk, cuda):
    # SPEC.md:327 random s.p.d. 7-banded pencils (6x6, 4x4) vs dense Kronecker solve;
    # SPEC.md:340 round trip: solve(apply_two_term(W)) == W
    rng = np.random.default_rng(327)

    def spd_band(k):
        B = np.tril(np.triu(rng.standard_normal((k, k)), -3), 3)
        S = B + B.T
        return S + (np.abs(S).sum(1).max() + 1) * np.eye(k)

    Mh, Qh, Mt, Qt = spd_band(6), spd_band(6), spd_band(4), spd_band(4)
    plan = plan_from_dense(stk, Mh, np.zeros((6, 6)), Qh, Qt, np.zeros((4, 4)), Mt)
    V = rng.standard_normal((4, 6))  # (nt, nh) == nh x nt column-major
    W = host(plan.two_term_solve(dev(V)))
    K = np.kron(Qt, Mh) + np.kron(Mt, Qh)  # vec(M W Qt^T + Q W Mt), Mt symmetric
    w = np.linalg.solve(K, V.ravel())
    assert rel(W.ravel(), w) < 1e-9
    Wr = rng.standard_normal((4, 6))
    back = host(plan.two_term_solve(plan.apply(dev(Wr))))  # A_h = 0: apply == two-term op
    assert rel(back, Wr) < 1e-9


def test_gmres_kats(stk, cuda):
    # SPEC.md:453 identity -> 1 iteration, x = b
    plan = plan_from_dense(stk, np.eye(5), np.zeros((5, 5)), np.zeros((5, 5)), np.eye(1),
                           np.zeros((1, 1)), np.zeros((1, 1)), precond=False)
    b = np.random.default_rng(3).standard_normal((1, 5))
    x, rep = plan.gmres(dev(b), stk.GmresConfig(tol=1e-12, maxit=10), precond=False)
    assert rep.iterations == 1 and rep.converged
    assert np.allclose(host(x), b, rtol=1e-15)
    # SPEC.md:454 diag(1..5), b = ones, no precond -> dense solve to 1e-10, <= 5 iterations
    plan = plan_from_dense(stk, np.diag(np.arange(1.0, 6.0)), np.zeros((5, 5)), np.zeros((5, 5)),
                           np.eye(1), np.zeros((1, 1)), np.zeros((1, 1)), precond=False)
    x, rep = plan.gmres(dev(np.ones((1, 5))), stk.GmresConfig(tol=1e-10, maxit=20), precond=False)
    assert rep.iterations <= 5 and rep.converged
    assert np.allclose(host(x).ravel(), 1.0 / np.arange(1.0, 6.0), rtol=1e-10)


@pytest.mark.parametrize("key", [("16_3", "16_3"), ("31_3", "33_3")])
def test_gmres_and_pcg_vs_oracle(stk, orc, ref_bands, cuda, key):
    sb, tb = ref_bands[f"space_{key[0]}"], ref_bands[f"time_{key[1]}"]
    plan = plan_from_bands(stk, sb, tb)
    W = orc.WaveSystemNP(sb, tb)
    rng = np.random.default_rng(7)
    b = rng.standard_normal(sb.shape[2] * tb.shape[2])
    xd = W.direct(b)
    x, rep = plan.gmres(dev(b), stk.GmresConfig(tol=1e-12, maxit=500))
    assert rep.converged
    hist = rep.rel_res_history
    assert all(h2 <= h1 * (1 + 1e-12) for h1, h2 in zip(hist, hist[1:]))
    xo, its, _ = W.gmres(b, tol=1e-12, maxit=500)
    assert abs(its - rep.iterations) <= 2  # same Krylov process (CGS2 vs MGS2 rounding)
    assert rel(host(x).ravel(), xd) < 1e-8
    assert rel(host(x).ravel(), xo) < 1e-8
    xp, rp = plan.pcg(dev(b), tol=1e-12, maxit=2000)
    assert rp.final_relres < 1e-10
    assert rel(host(xp).ravel(), xd) < 1e-8


def test_cfg4_pcg_and_gmres(stk, cuda):
    """Config 4 (1023 x 1025, N(0,1) F): PCG to the attainable floor, full GMRES for a fixed
    budget; both decrease the true residual monotonically and agree with each other."""
    from paper_1912_10082_b200 import inputs
    cfg = inputs.CONFIGS["cfg4"]
    sm = stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, cfg.nh))
    tm = stk.wave_time_matrices(stk.TimeGrid(cfg.nt, 1.0))
    plan = stk.WavePlan(sm, tm)
    F = dev(inputs.wave_rhs_host(cfg))
    x, rep = plan.pcg(F, tol=1e-9, maxit=6000)
    print("cfg4 PCG", rep.iterations, rep.final_relres, rep.wall_time_s)
    assert rep.final_relres < 1e-6  # measured FP64 floor is ~1e-7..1e-6
    xg, rg = plan.gmres(F, stk.GmresConfig(tol=1e-9, maxit=300))
    print("cfg4 GMRES(300)", rg.iterations, rg.final_relres, rg.wall_time_s)
    assert rg.final_relres < 1e-2
    hist = rg.rel_res_history
    assert all(h2 <= h1 * (1 + 1e-12) for h1, h2 in zip(hist, hist[1:]))


def test_generic_gmres_callback_seam(stk, ref_bands, cuda):
    """gmres over arbitrary VecOp callables (stk/outer_krylov.hpp:30,75) equals the plan path."""
    import torch
    sb, tb = ref_bands["space_16_3"], ref_bands["time_16_3"]
    plan = plan_from_bands(stk, sb, tb)
    b = dev(np.random.default_rng(9).standard_normal(sb.shape[2] * tb.shape[2]))
    cfg = stk.GmresConfig(tol=1e-11, maxit=300)
    x1, r1 = stk.gmres(stk.WaveOperator(plan), stk.TwoTermPrecond(plan), b, cfg)
    x2, r2 = stk.gmres(lambda v: plan.apply(v), lambda v: plan.two_term_solve(v), b, cfg)
    assert r1.iterations == r2.iterations and r2.converged
    assert torch.equal(x1, x2)
    # a plain diagonal operator through the callback seam (SPEC.md:454 analogue)
    d = torch.arange(1.0, 6.0, dtype=torch.float64, device="cuda")
    x, r = stk.gmres(lambda v: d * v, None, torch.ones(5, dtype=torch.float64, device="cuda"),
                     stk.GmresConfig(tol=1e-12, maxit=10))
    assert r.iterations <= 5 and torch.allclose(x, 1.0 / d, rtol=1e-12)


# ------------------------------------------- extended-precision residual and refinement --
def _longdouble_residual(orc, sb, tb, b, xh, xl):
    """b - B x in numpy longdouble (64-bit mantissa) with B from the raw bands."""
    L = np.longdouble
    dense = lambda band: orc.band_sparse(band).toarray().astype(L)
    Mh, Ah, Qh = (dense(sb[k]) for k in range(3))
    Qt, Dt, Mt = (dense(tb[k]) for k in range(3))
    E = Dt + Dt.T
    nh, nt = sb.shape[2], tb.shape[2]
    U = (xh.astype(L) + xl.astype(L)).reshape(nt, nh).T
    out = (Mh @ U) @ Qt.T + (Ah @ U) @ E + (Qh @ U) @ Mt
    r = b.astype(L) - out.T.ravel()
    return float(np.sqrt(np.sum(r * r)) / np.sqrt(np.sum(b.astype(L) ** 2)))


def test_residual_dd_vs_longdouble(stk, orc, ref_bands, cuda):
    """stkg_wave_residual_dd agrees with an independent 64-bit-mantissa evaluation, and both
    sit far below what the FP64 residual can resolve for a PCG iterate."""
    sb, tb = ref_bands["space_31_3"], ref_bands["time_33_3"]
    plan = plan_from_bands(stk, sb, tb)
    rng = np.random.default_rng(11)
    b = rng.standard_normal(plan.N)
    x, _ = plan.pcg(dev(b), tol=1e-12, maxit=3000)
    xh = host(x)
    xl = rng.standard_normal(plan.N) * 1e-20  # a genuine low part
    rel_dd = plan.residual_dd(dev(b), x, dev(xl))
    rel_ld = _longdouble_residual(orc, sb, tb, b, xh, xl)
    assert abs(rel_dd - rel_ld) <= 1e-3 * rel_ld + 1e-17


def test_refined_solve_small(stk, orc, ref_bands, cuda):
    sb, tb = ref_bands["space_31_3"], ref_bands["time_33_3"]
    plan = plan_from_bands(stk, sb, tb)
    b = np.random.default_rng(12).standard_normal(plan.N)
    xh, xl, rep = plan.solve_refined(dev(b), tol=1e-14, inner_tol=1e-6)
    assert rep.converged and rep.final_relres <= 1e-14
    assert _longdouble_residual(orc, sb, tb, b, host(xh), host(xl)) <= 1e-14
    h = rep.rel_res_history
    assert h[0] == 1.0 and all(b2 < b1 for b1, b2 in zip(h, h[1:]))


def test_cfg4_refined_to_north_star_tolerance(stk, cuda):
    """Config 4 to the north_star wave bar (1e-10), measured on the double-double residual:
    FP64 PCG alone stalls near 1e-7; two to three refinement rounds reach it."""
    from paper_1912_10082_b200 import inputs
    cfg = inputs.CONFIGS["cfg4"]
    sm = stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, cfg.nh))
    tm = stk.wave_time_matrices(stk.TimeGrid(cfg.nt, 1.0))
    plan = stk.WavePlan(sm, tm)
    F = dev(inputs.wave_rhs_host(cfg))
    xh, xl, rep = plan.solve_refined(F, tol=1e-10, inner_tol=1e-6, max_refine=6)
    print("cfg4 refined", rep.rel_res_history, rep.iterations, rep.wall_time_s)
    assert rep.converged and rep.final_relres <= 1e-10
    assert plan.residual_dd(F, xh, xl) <= 1e-10


def test_restarted_gmres(stk, ref_bands, cuda):
    """GmresConfig.restart > 0 (stk/outer_krylov.hpp:18-28): restarted cycles still reach the
    tolerance on the true residual, and the history has one entry per iteration."""
    sb, tb = ref_bands["space_16_3"], ref_bands["time_16_3"]
    plan = plan_from_bands(stk, sb, tb)
    b = dev(np.random.default_rng(21).standard_normal(plan.N))
    x, rep = plan.gmres(b, stk.GmresConfig(tol=1e-10, maxit=600, restart=15))
    assert rep.converged and rep.final_relres <= 1e-9
    assert len(rep.rel_res_history) == rep.iterations
    xf, repf = plan.gmres(b, stk.GmresConfig(tol=1e-10, maxit=600, restart=0))
    assert repf.iterations <= rep.iterations  # full GMRES never needs more iterations


# ------------------------------------------- space-modal time-banded preconditioner --
@pytest.mark.parametrize("key", [("16_3", "16_3"), ("31_3", "33_3")])
def test_modal_banded_solve_vs_oracle(stk, orc, ref_bands, cuda, key):
    """stkg_modal_banded_solve (2 DMMA GEMMs + a banded Cholesky solve per spatial mode)
    against the oracle's dense restatement (scipy eigh basis, dense s.p.d. solves)."""
    sb, tb = ref_bands[f"space_{key[0]}"], ref_bands[f"time_{key[1]}"]
    plan = plan_from_bands(stk, sb, tb)
    W = orc.WaveSystemNP(sb, tb)
    v = np.random.default_rng(21).standard_normal(plan.N)
    w = host(plan.modal_banded_solve(dev(v))).ravel()
    assert rel(w, W.modal_banded(v)) < 1e-9


def test_modal_banded_pcg_and_gmres(stk, orc, ref_bands, cuda):
    """With the modal banded preconditioner PCG and right-preconditioned GMRES converge in a
    size-independent ~10 iterations (TwoTermPrecond: 100s) to the direct solution."""
    sb, tb = ref_bands["space_31_3"], ref_bands["time_33_3"]
    plan = plan_from_bands(stk, sb, tb)
    W = orc.WaveSystemNP(sb, tb)
    b = np.random.default_rng(22).standard_normal(plan.N)
    xd = W.direct(b)
    plan.set_preconditioner("modal_banded")
    xp, rp = plan.pcg(dev(b), tol=1e-12, maxit=200)
    xg, rg = plan.gmres(dev(b), stk.GmresConfig(tol=1e-12, maxit=200))
    plan.set_preconditioner("two_term")
    _, r2 = plan.pcg(dev(b), tol=1e-12, maxit=3000)
    print("modal banded: pcg", rp.iterations, "gmres", rg.iterations, "| two-term pcg", r2.iterations)
    assert rp.converged and rg.converged and rp.iterations <= 25 and rg.iterations <= 25
    assert r2.iterations > 3 * rp.iterations
    assert rel(host(xp).ravel(), xd) < 1e-8 and rel(host(xg).ravel(), xd) < 1e-8


def test_cfg4_modal_banded_pcg_and_refined(stk, cuda):
    """Config 4 with the modal banded preconditioner: PCG to 1e-7 in <= 30 iterations
    (TwoTermPrecond: 1370), and the refined solve to the north_star 1e-10 bar."""
    from paper_1912_10082_b200 import inputs
    cfg = inputs.CONFIGS["cfg4"]
    sm = stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, cfg.nh))
    tm = stk.wave_time_matrices(stk.TimeGrid(cfg.nt, 1.0))
    plan = stk.WavePlan(sm, tm, preconditioner="modal_banded")
    F = dev(inputs.wave_rhs_host(cfg))
    x, rep = plan.pcg(F, tol=1e-7, maxit=500)
    print("cfg4 modal banded pcg", rep.iterations, rep.final_relres, rep.wall_time_s)
    assert rep.converged and rep.iterations <= 30 and rep.final_relres <= 2e-7
    xh, xl, rr = plan.solve_refined(F, tol=1e-10, inner_tol=1e-6, max_refine=6)
    print("cfg4 modal banded refined", rr.rel_res_history, rr.iterations, rr.wall_time_s)
    assert rr.converged and plan.residual_dd(F, xh, xl) <= 1e-10


@pytest.mark.parametrize("nh,nt", [(63, 256), (127, 128), (40, 400)])
def test_modal_banded_chunked_substitution_vs_oracle(stk, orc, cuda, nh, nt):
    """The parallel-in-time banded substitution (16 or 8 time chunks per mode with 3 x 3
    chunk transfers, n_t >= 256 / 128) against the oracle's dense restatement."""
    sm = stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, nh))
    tm = stk.wave_time_matrices(stk.TimeGrid(nt, 1.0))
    sb = np.stack([sm.M.band, sm.A.band, sm.Q.band])
    tb = np.stack([tm.Q.band, tm.D.band, tm.M.band])
    plan = stk.WavePlan(sm, tm)
    W = orc.WaveSystemNP(sb, tb)
    v = np.random.default_rng(nh + nt).standard_normal(plan.N)
    w = host(plan.modal_banded_solve(dev(v))).ravel()
    # agreement with the dense restatement is limited by cond(K_i): ~3.5e9 for the lowest
    # spatial mode at n_t = 256, where two backward-stable solvers differ by ~1e-9 (and the
    # FP64 evaluation of P w is no sharper); the Krylov solves' true residuals are the
    # accuracy check that matters (test_modal_banded_pcg_and_gmres, cfg4 test)
    assert rel(w, W.modal_banded(v)) < 1e-7


_SK_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1912_10082_b200 as stk
sm = stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, 300))
tm = stk.wave_time_matrices(stk.TimeGrid(320, 1.0))
plan = stk.WavePlan(sm, tm)
v = torch.from_numpy(np.random.default_rng(5).standard_normal(plan.N)).cuda()
out = {"tt": plan.two_term_solve(v).cpu().numpy(), "mb": plan.modal_banded_solve(v).cpu().numpy()}
np.savez(sys.argv[2], **out)
"""


def test_streamk_gemm_matches_default(tmp_path):
    """The opt-in stream-K GEMM schedule (STKG_STREAMK=1: split tiles finished by their first
    segment's CTA, later segments' partials added in fixed order) gives the preconditioner
    products of the one-tile-per-CTA kernel to rounding."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    res = {}
    for v in ("1", "0"):
        f = tmp_path / f"sk{v}.npz"
        subprocess.run([sys.executable, "-c", _SK_SCRIPT, root, str(f)], check=True,
                       env=dict(os.environ, STKG_STREAMK=v))
        res[v] = dict(np.load(f))
    for k in res["0"]:
        assert rel(res["1"][k], res["0"][k]) < 1e-12, k
