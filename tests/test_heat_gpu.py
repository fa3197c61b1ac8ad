"""GPU parity tests of the heat hot path (K1 operator/residual, K2 DMMA transforms, K3 scan)
against the CPU oracle, through the C ABI (ctypes binding in paper_1912_10082_b200)."""
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


def p1_setup(stk, ndim, n, nt, T=1.0):
    g = stk.SpaceGrid1D(0.0, 1.0, n)
    M, A = stk.fem1d_matrices(g)
    D, Cm = stk.heat_time_matrices(stk.TimeGrid(nt, T))
    eig = stk.TensorEigPair([stk.p1_eigpair(g)] * ndim)
    plan = stk.HeatPlan(eig, D, Cm, [M] * ndim, [A] * ndim)
    return plan, M, A, D, Cm


def orc_factors(stk_m, stk_a, D, Cm, ndim):
    m = (stk_m.diag, stk_m.off)
    a = (stk_a.diag, stk_a.off)
    return [m] * ndim, [a] * ndim, (D.diag, D.sup), (Cm.diag, Cm.sup)


# ------------------------------------------------------------- K2+K3 vs dense oracle --
@pytest.mark.parametrize("ns,nt", [((1,), 1), ((3,), 5), ((37,), 11), ((130,), 33), ((257,), 7),
                                   ((5, 7), 9), ((17, 13), 4), ((3, 4, 5), 6), ((1, 9, 2), 3)])
def test_solve_random_tensor_eigpair_vs_dense_oracle(stk, orc, cuda, ns, nt):
    """solve_projected_heat_with with an arbitrary (non-orthogonal) tensor EigPair: the GPU
    tensor-form transforms + scan equal the oracle's dense k x k restatement."""
    rng = np.random.default_rng(sum(ns) * 31 + nt)
    axes, Xs, lams = [], [], []
    for n in ns:
        X = rng.standard_normal((n, n)) / np.sqrt(n)
        lam = rng.uniform(0.5, 50.0, n)
        axes.append(stk.EigPair(lam, X))
        Xs.append(X)
        lams.append(lam)
    Xk = Xs[0]
    lk = lams[0]
    for X, lam in zip(Xs[1:], lams[1:]):
        Xk = np.kron(Xk, X)  # index ix*ny + iy (sparse_kron order)
        lk = (lk[:, None] + lam[None, :]).ravel()
    D, Cm = stk.heat_time_matrices(stk.TimeGrid(nt, 1.0))
    F = rng.standard_normal((nt, Xk.shape[0]))
    plan = stk.HeatPlan(stk.TensorEigPair(axes), D, Cm)
    U = host(plan.solve(dev(F)))
    Uref = orc.solve_projected_heat_with_dense(Xk, lk, (D.diag, D.sup), (Cm.diag, Cm.sup), F)
    assert rel(U, Uref) < 1e-12


def test_kat_scalar_and_diag(stk, orc, cuda):
    # SPEC.md:307  k=1, N_t=1, h_m=d=1, h_a=c=1, g=2 -> y=1
    one = stk.Bidiagonal(np.array([1.0]), np.zeros(0))
    plan = stk.HeatPlan(stk.EigPair(np.array([1.0]), np.array([[1.0]])), one, one)
    assert host(plan.solve(dev([[2.0]])))[0, 0] == 1.0
    # SPEC.md:308  H_M = I, H_A = diag(1,2), heat D,C with N_t=3, dt=1, G = ones
    D, Cm = stk.heat_time_matrices(stk.TimeGrid(3, 3.0))
    plan = stk.HeatPlan(stk.EigPair(np.array([1.0, 2.0]), np.eye(2)), D, Cm)
    Y = host(plan.solve(dev(np.ones((3, 2)))))
    B = np.kron(D.dense().T, np.eye(2)) + np.kron(Cm.dense().T, np.diag([1.0, 2.0]))
    assert np.allclose(Y.ravel(), np.linalg.solve(B, np.ones(6)), rtol=1e-14, atol=1e-15)


def test_kat_random_spd_residual(stk, cuda):
    # SPEC.md:309  random s.p.d. H_M, H_A (k=5), N_t=7 -> residual <= 1e-11 relative
    rng = np.random.default_rng(309)
    B1 = rng.standard_normal((5, 5))
    B2 = rng.standard_normal((5, 5))
    HM = B1 @ B1.T + 5 * np.eye(5)
    HA = B2 @ B2.T + np.eye(5)
    eig = stk.sym_gen_eig(HA, HM)
    D, Cm = stk.heat_time_matrices(stk.TimeGrid(7, 1.0))
    G = rng.standard_normal((7, 5))
    Y = host(stk.HeatPlan(eig, D, Cm).solve(dev(G)))
    R = HM @ Y.T @ D.dense() + HA @ Y.T @ Cm.dense() - G.T
    assert np.linalg.norm(R) / np.linalg.norm(G) <= 1e-11


def test_singular_row_system_raises(stk, cuda):
    # stk/sylvester.hpp:133-135: |d_j + lambda c_j| < 1e-300 -> SingularityError
    D = stk.Bidiagonal(np.array([1.0, 0.0]), np.array([-1.0]))
    Cm = stk.Bidiagonal(np.array([0.5, 0.0]), np.array([0.5]))
    plan = stk.HeatPlan(stk.EigPair(np.array([2.0]), np.array([[1.0]])), D, Cm)
    with pytest.raises(stk.SingularityError, match="lambda"):
        plan.solve(dev(np.ones((2, 1))))


# ------------------------------------------------------------------------ K1 apply ---
@pytest.mark.parametrize("ndim,n,nt", [(1, 1, 1), (1, 40, 9), (2, 1, 3), (2, 11, 6),
                                       (2, 63, 17), (3, 5, 4), (3, 12, 5)])
def test_apply_vs_oracle(stk, orc, cuda, ndim, n, nt):
    plan, M, A, D, Cm = p1_setup(stk, ndim, n, nt)
    ms, as_, d, c = orc_factors(M, A, D, Cm, ndim)
    rng = np.random.default_rng(n * 7 + nt)
    U = rng.standard_normal((nt, n ** ndim))
    Y = host(plan.apply(dev(U)))
    Yref = orc.heat_apply(ms, as_, d, c, U)
    assert rel(Y, Yref) < 1e-13


def test_apply_linearity_and_residual(stk, orc, cuda):
    # SPEC.md:339 linearity; residual == ||F - B(U)|| / ||F||
    plan, M, A, D, Cm = p1_setup(stk, 2, 21, 8)
    rng = np.random.default_rng(2)
    X, Y = rng.standard_normal((2, 8, 441))
    a, b = 0.3, -1.7
    lhs = host(plan.apply(dev(a * X + b * Y)))
    rhs = a * host(plan.apply(dev(X))) + b * host(plan.apply(dev(Y)))
    assert rel(lhs, rhs) < 1e-14
    F = rng.standard_normal((8, 441))
    r_gpu, fn = plan.residual(dev(X), dev(F))
    ms, as_, d, c = orc_factors(M, A, D, Cm, 2)
    assert abs(fn - np.linalg.norm(F)) < 1e-12 * fn
    assert abs(r_gpu - orc.heat_residual(ms, as_, d, c, X, F)) < 1e-13


# ---------------------------------------------------------------- BASELINE configs ---
def _config_parity(stk, orc, name, nsteps=None, cn_steps=None):
    from paper_1912_10082_b200 import inputs
    cfg = inputs.CONFIGS[name]
    plan, M, A, D, Cm = p1_setup(stk, cfg.ndim, cfg.n, cfg.nt)
    ms, as_, d, c = orc_factors(M, A, D, Cm, cfg.ndim)
    if cfg.rank == 0:
        Fd = inputs.heat_rhs_device(cfg)
        Fh = inputs.heat_rhs_host(cfg, nsteps=nsteps)
        assert np.array_equal(host(Fd[: Fh.shape[0]]), Fh)  # device generator == host
    else:
        Fh_full = inputs.heat_rhs_host(cfg)
        Fd = dev(Fh_full)
        Fh = Fh_full if nsteps is None else Fh_full[:nsteps]
    U = plan.solve(Fd)
    relres, _ = plan.residual(U, Fd)
    assert relres <= 1e-10, relres  # north_star gate, checked by the GPU residual kernel
    eig = orc.p1_pencil_eig(ms[0], as_[0])  # scipy eigh basis: independent of the closed form
    Uref = orc.heat_decoupled([eig] * cfg.ndim, d, c, Fh, nsteps=nsteps)
    k = Uref.shape[0]
    err = rel(host(U[:k]), Uref)
    assert err <= 1e-10, err
    if cn_steps:
        Ucn = orc.crank_nicolson(ms, as_, 1.0 / cfg.nt, Fh, nsteps=cn_steps)
        assert rel(host(U[:cn_steps]), Ucn) <= 1e-10
    return relres, err


def test_cfg1_parity(stk, orc, cuda):
    _config_parity(stk, orc, "cfg1", cn_steps=256)


def test_cfg2_parity(stk, orc, cuda):
    _config_parity(stk, orc, "cfg2", cn_steps=16)


def test_cfg5_parity(stk, orc, cuda):
    _config_parity(stk, orc, "cfg5", nsteps=16)


def test_cfg3_parity_prefix_and_full_residual(stk, orc, cuda):
    # full 1023^2 x 1024 solve on the GPU; causal 8-step prefix vs the numpy oracle (the
    # first k columns of U depend only on the first k columns of F), full-size residual.
    _config_parity(stk, orc, "cfg3", nsteps=8)


# ------------------------------------------------------------ host path / determinism --
def test_host_path_bitwise_equal_device_path(stk, cuda):
    import torch
    plan, *_ = p1_setup(stk, 2, 63, 40)
    eig = stk.TensorEigPair([stk.p1_eigpair(stk.SpaceGrid1D(0, 1, 63))] * 2)
    D, Cm = stk.heat_time_matrices(stk.TimeGrid(40, 1.0))
    plan_c = stk.HeatPlan(eig, D, Cm, time_chunk=7)
    rng = np.random.default_rng(11)
    F = rng.standard_normal((40, 63 * 63))
    Ud = host(plan.solve(dev(F)))
    Uh = plan_c.solve_host(F)  # 6 chunks of 7 steps (+ remainder), carry across chunks
    assert np.array_equal(Ud, Uh)
    pinned = torch.from_numpy(F).pin_memory()
    out = torch.empty_like(pinned).pin_memory()
    plan_c.solve_host(pinned.numpy(), out=out.numpy())
    assert np.array_equal(out.numpy(), Ud)
    # determinism: same inputs -> bit-identical solution and residual
    assert np.array_equal(host(plan.solve(dev(F))), Ud)
    r1 = plan.residual(dev(Ud), dev(F))
    r2 = plan.residual(dev(Ud), dev(F))
    assert r1 == r2


@pytest.mark.parametrize("ndim,n,nt,rank", [(1, 255, 256, 1), (2, 63, 40, 4), (3, 15, 12, 8),
                                            (2, 17, 9, 16)])
def test_factored_load_equals_dense_load(stk, orc, cuda, ndim, n, nt, rank):
    """F = L R^T solved from its factors equals the dense-F solve and the oracle."""
    plan, M, A, D, Cm = p1_setup(stk, ndim, n, nt)
    rng = np.random.default_rng(rank)
    L = rng.standard_normal((rank, n ** ndim))  # == n_x x rank column-major
    R = rng.standard_normal((rank, nt))
    F = R.T @ L  # (nt, n_x) == L R^T column-major
    Uf = host(plan.solve_factored(dev(L), dev(R)))
    Ud = host(plan.solve(dev(F)))
    assert rel(Uf, Ud) < 1e-13
    ms, as_, d, c = orc_factors(M, A, D, Cm, ndim)
    Uref = orc.heat_decoupled([orc.p1_pencil_eig(ms[0], as_[0])] * ndim, d, c, F)
    assert rel(Uf, Uref) < 1e-10


# --------------------------------------------------------------- fast sine transforms --
@pytest.mark.parametrize("ndim,n,nt", [(1, 15, 7), (1, 255, 256), (2, 15, 5), (2, 63, 17),
                                       (2, 127, 4), (3, 15, 6), (3, 31, 3), (1, 2047, 3),
                                       (2, 1023, 2), (1, 511, 9), (2, 511, 3), (3, 511, 1),
                                       (2, 2047, 1), (1, 1023, 5), (2, 255, 4), (3, 127, 2),
                                       (2, 31, 3), (3, 63, 1),
                                       # few modes, long time axes: the chunked parallel-in-time
                                       # scan (registers for n_t <= 512, re-read beyond)
                                       (1, 127, 1100), (2, 31, 700), (2, 63, 333), (1, 15, 31)])
def test_dst_backend_equals_dense_backend(stk, cuda, ndim, n, nt):
    """The P1 fast-sine-transform backend computes the same solve_projected_heat_with as the
    dense DMMA backend on the closed-form eigenbasis (X = S diag(mu^-1/2))."""
    rng = np.random.default_rng(n + nt)
    F = rng.standard_normal((nt, n ** ndim))
    pd = stk.HeatPlan.p1_uniform(ndim, n, nt, transform="dense")
    ps = stk.HeatPlan.p1_uniform(ndim, n, nt, transform="dst")
    Ud = host(pd.solve(dev(F)))
    Us = host(ps.solve(dev(F)))
    # the half-length DST's odd outputs are a prefix sum over k, whose rounding grows like
    # sqrt(N) eps (dst_half.cuh): ~1e-13 at N = 2048 instead of ~1e-14
    assert rel(Us, Ud) < (1e-12 if n < 511 else 2e-12), rel(Us, Ud)
    rr, _ = ps.residual(dev(Us), dev(F))
    print(ndim, n, nt, "rel vs dense", rel(Us, Ud), "relres", rr)
    assert rr < 1e-10  # north_star gate (cond grows ~ n^2: 3e-12 at n = 2047, nt = 3)


@pytest.mark.parametrize("name,nsteps", [("cfg1", None), ("cfg2", None), ("cfg5", 16), ("cfg3", 8)])
def test_dst_config_parity(stk, orc, cuda, name, nsteps):
    """BASELINE configs through the fast-sine-transform backend: GPU relres and the oracle."""
    from paper_1912_10082_b200 import inputs
    cfg = inputs.CONFIGS[name]
    plan = stk.HeatPlan.p1_uniform(cfg.ndim, cfg.n, cfg.nt, transform="dst")
    if cfg.rank == 0:
        Fd = inputs.heat_rhs_device(cfg)
        Fh = inputs.heat_rhs_host(cfg, nsteps=nsteps)
    else:
        Fh_full = inputs.heat_rhs_host(cfg)
        Fd = dev(Fh_full)
        Fh = Fh_full if nsteps is None else Fh_full[:nsteps]
    U = plan.solve(Fd)
    relres, _ = plan.residual(U, Fd)
    assert relres <= 1e-10, relres
    m, a = orc.fem1d_matrices(0.0, 1.0, cfg.n)
    d, c = orc.heat_time_matrices(cfg.nt)
    Uref = orc.heat_decoupled([orc.p1_pencil_eig(m, a)] * cfg.ndim, d, c, Fh, nsteps=nsteps)
    assert rel(host(U[: Uref.shape[0]]), Uref) <= 1e-10


def test_dst_host_and_factored_paths(stk, cuda):
    ps = stk.HeatPlan.p1_uniform(2, 63, 40, transform="dst", time_chunk=7)
    rng = np.random.default_rng(5)
    L = rng.standard_normal((3, 63 * 63))
    R = rng.standard_normal((3, 40))
    F = R.T @ L
    Ud = host(ps.solve(dev(F)))
    # two real vectors share one complex FFT; time chunking changes the pairing, so the
    # host-buffer path agrees to rounding (not bitwise) in this backend
    assert rel(ps.solve_host(F), Ud) < 1e-14
    assert np.array_equal(host(ps.solve(dev(F))), Ud)  # deterministic
    assert rel(host(ps.solve_factored(dev(L), dev(R))), Ud) < 1e-13


# ------------------------------------------------------------------------------ RKSM --
def _smooth_load(n, ndim, nt, T=1.0):
    """heat-ex1-shaped separable load (stk/bench.hpp:302-306): 10 sin(t) t x cos(pi x/2)^ndim,
    lumped onto the P1 basis (midpoint in time)."""
    h = 1.0 / (n + 1)
    f = np.cos(np.pi / 2 * np.arange(1, n + 1) * h) * h
    L = f
    for _ in range(ndim - 1):
        L = np.kron(L, f)
    tt = (np.arange(nt) + 0.5) * T / nt
    return L[None, :], (10 * np.sin(tt) * tt * T / nt)[None, :]


def _rksm_oracle(orc, ndim, n, nt, L, R, **kw):
    m, a = orc.fem1d_matrices(0.0, 1.0, n)
    d, c = orc.heat_time_matrices(nt)
    left, right, its, hist = orc.rksm_solve([m] * ndim, [a] * ndim, d, c, L.T, R.T, **kw)
    return (left @ right.T).T, its, hist


def _rksm_gpu(stk, ndim, n, nt, L, R, transform="dense", **kw):
    plan = stk.HeatPlan.p1_uniform(ndim, n, nt, transform=transform)
    UL, UR, rep = plan.rksm(dev(L), dev(R), **kw)
    return plan, host(UR).T @ host(UL), rep


@pytest.mark.parametrize("n,nt,rank,src", [(10, 6, 1, "rand"), (63, 40, 3, "rand"),
                                           (255, 256, 1, "cfg1"), (255, 256, 1, "smooth")])
def test_rksm_1d_converges_vs_oracle_and_direct(stk, orc, cuda, n, nt, rank, src):
    """rksm_solve (stk/rksm.hpp:127-234), 1D (shifted solves = batched Thomas): converges to
    1e-8; the truncated solution matches the direct solve to 1e-6 (SPEC.md:411 example,
    cfg1's shape) and the oracle's iterate and iteration count."""
    from paper_1912_10082_b200 import inputs
    if src == "cfg1":
        left, right = inputs.heat_factors(inputs.CONFIGS["cfg1"])
        L, R = left.T.copy(), right.T.copy()
    elif src == "smooth":
        L, R = _smooth_load(n, 1, nt)
    else:
        rng = np.random.default_rng(n)
        L, R = rng.standard_normal((rank, n)), rng.standard_normal((rank, nt))
    plan, U, rep = _rksm_gpu(stk, 1, n, nt, L, R, tol=1e-8, maxit=100)
    assert rep.converged and rep.final_relres <= 1e-8
    assert len(rep.rel_res_history) == rep.iterations
    Ud = host(plan.solve_factored(dev(L), dev(R)))
    assert rel(U, Ud) <= 1e-6
    rr, _ = plan.residual(dev(U), dev(R.T @ L))
    assert rr <= 1e-5  # truncation at tol perturbs U by 1e-8 ||U||; B amplifies it
    Uo, its, hist = _rksm_oracle(orc, 1, n, nt, L, R, tol=1e-8, maxit=100)
    assert abs(its - rep.iterations) <= 1
    assert rel(U, Uo) <= 1e-6


@pytest.mark.parametrize("transform,ndim,n,nt", [("dense", 2, 31, 20), ("dst", 2, 31, 20),
                                                 ("dense", 3, 15, 12), ("dst", 3, 15, 12)])
def test_rksm_2d_history_vs_oracle(stk, orc, cuda, transform, ndim, n, nt):
    """2D, fixed_iters (preconditioner mode, stk/rksm.hpp:172,226): per-iteration relative
    residuals and the truncated iterate follow the oracle.  (With real negative poles the
    reference's adaptive rule stalls near 1e-4 on 2D heat loads -- see DESIGN.md -- so
    2D parity is on the history, not on convergence.)"""
    L, R = _smooth_load(n, ndim, nt)
    rng = np.random.default_rng(5)
    L = np.vstack([L, rng.standard_normal((1, n ** ndim))])
    R = np.vstack([R, rng.standard_normal((1, nt))])
    _, U, rep = _rksm_gpu(stk, ndim, n, nt, L, R, transform=transform, fixed_iters=8)
    Uo, its, hist = _rksm_oracle(orc, ndim, n, nt, L, R, fixed_iters=8)
    assert rep.iterations == its == 8 and rep.converged
    np.testing.assert_allclose(rep.rel_res_history, hist, rtol=1e-6)
    assert rel(U, Uo) <= 1e-8


def test_rksm_maxit_and_zero_load(stk, orc, cuda):
    """maxit reached above tol -> non-convergence result with the full history
    (stk/rksm.hpp:201-204); F = 0 -> rank 0, 0 iterations (:137-141)."""
    n, nt = 31, 24
    L, R = _smooth_load(n, 2, nt)
    _, U, rep = _rksm_gpu(stk, 2, n, nt, L, R, tol=1e-12, maxit=12)
    assert not rep.converged and rep.iterations == 12 and len(rep.rel_res_history) == 12
    Uo, its, hist = _rksm_oracle(orc, 2, n, nt, L, R, tol=1e-12, maxit=12)
    np.testing.assert_allclose(rep.rel_res_history, hist, rtol=1e-6)
    assert rel(U, Uo) <= 1e-8
    _, U0, rep0 = _rksm_gpu(stk, 2, n, nt, np.zeros((1, n * n)), np.ones((1, nt)))
    assert rep0.iterations == 0 and rep0.rank == 0 and rep0.converged and not U0.any()


def test_rksm_cfg2_shape(stk, cuda):
    """BASELINE cfg2 shape (2D 255^2 x 512, rank-4 N(0,1) load): both transform backends give
    the same history; the true residual of the returned factors equals the reported one."""
    from paper_1912_10082_b200 import inputs
    cfg = inputs.CONFIGS["cfg2"]
    left, right = inputs.heat_factors(cfg)
    L, R = left.T.copy(), right.T.copy()
    out = {}
    for transform in ("dst", "dense"):
        plan, U, rep = _rksm_gpu(stk, 2, cfg.n, cfg.nt, L, R, transform=transform, maxit=15)
        rr, _ = plan.residual(dev(U), dev(R.T @ L))
        assert abs(rr - rep.final_relres) <= 1e-6 * max(rr, 1e-12) + 1e-9
        out[transform] = rep.rel_res_history
        print(transform, "its", rep.iterations, "relres", rep.final_relres, "s", rep.wall_time_s)
    np.testing.assert_allclose(out["dst"], out["dense"], rtol=1e-6)


# --- the reference's own RKSM acceptance problems ---------------------
@pytest.mark.parametrize("ndim,nh", [(1, 199), (2, 60), (3, 24)])
def test_rksm_heat_ex1_acceptance(stk, orc, cuda, ndim, nh):
    """rksm_solve on the reference's heat-ex1 desk problem (stk/bench.hpp:300-306,361-406:
    Omega=(-1,1)^d, T=10, load 10 sin(t) t prod cos(pi x_i/2) projected by project_rhs_heat,
    stk/rhs_sep.hpp:111-151), N_t in {100, 300, 500}, GPU and oracle both:
    SPEC.md:614-615 -- iterations <= 30 with spread <= 3, rank <= 20, mu_mem <= 40 (the 2D
    60 x 60 problem; 1D and 3D the same problem on other axes counts); SPEC.md:613 -- in 1D
    (N_h=199, trapezoidal-time RHS) the space-time solution equals the CN trajectory column
    by column to 1e-6.  The GPU iterate also matches the oracle's and the direct solve.
    (n+1 is not a power of two here, so the plan uses the dense DMMA transforms.)"""
    its_all = []
    for nt in (100, 300, 500):
        L, H = orc.heat_ex1_load(ndim, nh, nt, T=10.0, trapezoidal_time=(ndim == 1))
        plan = stk.HeatPlan.p1_uniform(ndim, nh, nt, T=10.0, a=-1.0, b=1.0, transform="dense")
        UL, UR, rep = plan.rksm(dev(L[None, :]), dev(H[None, :]), tol=1e-8, maxit=60)
        U = host(UR).T @ host(UL)
        assert rep.converged and rep.final_relres <= 1e-8
        assert rep.iterations <= 30 and rep.rank <= 20 and rep.mu_mem <= 40, rep
        its_all.append(rep.iterations)
        m, a = orc.fem1d_matrices(-1.0, 1.0, nh)
        d, c = orc.heat_time_matrices(nt, 10.0)
        left, right, its, hist = orc.rksm_solve([m] * ndim, [a] * ndim, d, c, L[:, None],
                                                H[:, None], tol=1e-8, maxit=60)
        assert its == rep.iterations
        Uo = (left @ right.T).T
        assert rel(U, Uo) <= 1e-6
        Ud = host(plan.solve_factored(dev(L[None, :]), dev(H[None, :])))
        assert rel(U, Ud) <= 1e-6
        if ndim == 1:
            Ucn = orc.crank_nicolson_splu([m], [a], 10.0 / nt, np.outer(H, L))
            col = np.linalg.norm(U - Ucn, axis=1) / np.linalg.norm(Ucn, axis=1)
            assert col.max() <= 1e-6, col.max()
    assert max(its_all) - min(its_all) <= 3


@pytest.mark.parametrize("seed", range(20))
def test_rksm_random_spd_pencils_vs_dense(stk, orc, cuda, seed):
    """SPEC.md:612 (criterion 1): 20 random heat instances, N_h <= 40, N_t <= 30, 1D FEM
    matrices plus random s.p.d. (tridiagonal, diagonally dominant) perturbations: rksm_solve
    at tol 1e-8 matches the dense solve of the (D^T (x) M + C^T (x) A) system to 1e-6."""
    rng = np.random.default_rng(1000 + seed)
    nh, nt, r = int(rng.integers(4, 41)), int(rng.integers(2, 31)), int(rng.integers(1, 4))
    g = stk.SpaceGrid1D(0.0, 1.0, nh)
    M, A = stk.fem1d_matrices(g)

    def perturb(t, scale):
        off = scale * rng.uniform(-1, 1, nh - 1)
        diag = scale * rng.uniform(0.1, 1.0, nh)
        diag[:-1] += np.abs(off)
        diag[1:] += np.abs(off)
        return stk.Tridiagonal(t.diag + diag, t.off + off)

    Mp = perturb(M, 0.1 * M.diag[0])
    Ap = perturb(A, 0.1 * A.diag[0])
    eig = stk.sym_gen_eig(Ap.dense(), Mp.dense())
    D, Cm = stk.heat_time_matrices(stk.TimeGrid(nt, 1.0))
    plan = stk.HeatPlan(eig, D, Cm, [Mp], [Ap], transform="dense")
    L, R = rng.standard_normal((r, nh)), rng.standard_normal((r, nt))
    UL, UR, rep = plan.rksm(dev(L), dev(R), tol=1e-8, maxit=100)
    assert rep.converged and rep.final_relres <= 1e-8
    U = host(UR).T @ host(UL)  # (nt, nh)
    K = np.kron(D.dense().T, Mp.dense()) + np.kron(Cm.dense().T, Ap.dense())
    u = np.linalg.solve(K, (L.T @ R).reshape(-1, order="F")).reshape(nh, nt, order="F")
    assert rel(U, u.T) <= 1e-6


def test_caller_buffers_are_size_checked_and_stream_ordered(stk, cuda):
    """Caller-provided outputs are size-checked before the C ABI writes them (host and
    device), and a plan call made under another torch stream is ordered with that stream's
    queued work (inputs written there are read after the writes; outputs are ready there)."""
    import torch
    plan = stk.HeatPlan.p1_uniform(2, 63, 8)
    F = torch.randn(8, 63 * 63, dtype=torch.float64, device="cuda")
    with pytest.raises(stk.ArgumentError):
        plan.solve_host(np.ones((8, 63 * 63)), out=np.empty((4, 63 * 63)))
    with pytest.raises(stk.ArgumentError):
        plan.apply(F, out=torch.empty(7, 63 * 63, dtype=torch.float64, device="cuda"))
    ref = host(plan.solve(F))
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        torch.cuda._sleep(50_000_000)  # keep the side stream busy before it writes F
        F2 = F * 1.0
        U = plan.solve(F2)
        got = U.clone()
    side.synchronize()
    np.testing.assert_array_equal(host(got), ref)


@pytest.mark.parametrize("ns,nt", [((63, 31), 5), ((15, 127), 3), ((31, 15, 63), 2), ((1023, 255), 2)])
def test_dst_mixed_axis_lengths(stk, cuda, ns, nt):
    """Different grid sizes per axis (each axis its own sine transform length, padded or
    half-length kernels mixed in one plan) against the dense DMMA backend."""
    grids = [stk.SpaceGrid1D(0.0, 1.0, n) for n in ns]
    eigs = [stk.p1_eigpair(g) for g in grids]
    mats = [stk.fem1d_matrices(g) for g in grids]
    D, Cm = stk.heat_time_matrices(stk.TimeGrid(nt, 1.0))
    ms, as_ = [m for m, _ in mats], [a for _, a in mats]
    pd = stk.HeatPlan(stk.TensorEigPair(eigs), D, Cm, ms, as_, transform="dense")
    ps = stk.HeatPlan(stk.TensorEigPair(eigs), D, Cm, ms, as_, transform="dst",
                      p1_h=[g.fem_h for g in grids])
    F = np.random.default_rng(sum(ns)).standard_normal((nt, int(np.prod(ns))))
    Ud, Us = host(pd.solve(dev(F))), host(ps.solve(dev(F)))
    assert rel(Us, Ud) < 2e-12
    rr, _ = ps.residual(dev(Us), dev(F))
    assert rr < 1e-10


@pytest.mark.parametrize("transform", ["dense", "dst"])
def test_nonuniform_time_bidiagonals(stk, orc, cuda, transform):
    """General (non-uniform) temporal bidiagonals D, C: the recurrence uses every step's own
    coefficients (stk/sylvester.hpp:128-140); both backends against the dense oracle."""
    rng = np.random.default_rng(17)
    n, nt = 31, 9
    g = stk.SpaceGrid1D(0.0, 1.0, n)
    e = stk.p1_eigpair(g)
    M, A = stk.fem1d_matrices(g)
    D = stk.Bidiagonal(rng.uniform(1.0, 2.0, nt), rng.uniform(-1.0, -0.2, nt - 1))
    Cm = stk.Bidiagonal(rng.uniform(0.01, 0.1, nt), rng.uniform(0.01, 0.1, nt - 1))
    kw = dict(transform=transform)
    if transform == "dst":
        kw["p1_h"] = [g.fem_h] * 2
    plan = stk.HeatPlan(stk.TensorEigPair([e, e]), D, Cm, [M, M], [A, A], **kw)
    F = rng.standard_normal((nt, n * n))
    U = host(plan.solve(dev(F)))
    rr, _ = plan.residual(dev(U), dev(F))
    assert rr < 1e-12
    Xk = np.kron(e.X, e.X)
    lk = (e.lambdas[:, None] + e.lambdas[None, :]).ravel()
    Uref = orc.solve_projected_heat_with_dense(Xk, lk, (D.diag, D.sup), (Cm.diag, Cm.sup), F)
    assert rel(U, Uref) < 1e-12


_PAD_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1912_10082_b200 as stk
out = {}
for ndim, n, nt in [(2, 1023, 3), (2, 255, 5), (3, 127, 3), (3, 63, 2), (2, 15, 4)]:
    F = torch.from_numpy(np.random.default_rng(n + ndim).standard_normal((nt, n ** ndim))).cuda()
    p = stk.HeatPlan.p1_uniform(ndim, n, nt, transform="dst")
    out[f"u{ndim}_{n}"] = p.solve(F).cpu().numpy()
    L = torch.from_numpy(np.random.default_rng(n).standard_normal((2, n ** ndim))).cuda()
    R = torch.from_numpy(np.random.default_rng(nt).standard_normal((2, nt))).cuda()
    out[f"f{ndim}_{n}"] = p.solve_factored(L, R).cpu().numpy()
np.savez(sys.argv[2], **out)
"""


def test_padded_layout_equals_unpadded(tmp_path):
    """The device solve's padded internal layout (fastest axis at pitch N, 16-byte strided
    kernel in place) computes what the unpadded passes compute.  Not bit for bit: two real
    vectors share one complex FFT, and the layouts pair different vectors (vector n - 1
    pairs with the zero pad lane instead of the next line's vector 0), so the partners'
    rounding differs.  Each layout runs in its own process (STKG_PAD is read once)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    res = {}
    for pad in ("1", "0"):
        f = tmp_path / f"pad{pad}.npz"
        # (both with the transform-based passes: this test is about the layout)
        env = dict(os.environ, STKG_PAD=pad, STKG_TRIDIAG="0")
        subprocess.run([sys.executable, "-c", _PAD_SCRIPT, root, str(f)], check=True, env=env)
        res[pad] = dict(np.load(f))
    for k in res["1"]:
        assert rel(res["1"][k], res["0"][k]) < 1e-13, (k, rel(res["1"][k], res["0"][k]))


def test_tma_strided_variant_matches(tmp_path):
    """The opt-in TMA staging of the strided DST pass (STKG_TMA=1: SWIZZLE_64B boxes into the
    same swizzled row mirror) computes bit for bit what the cp.async staging computes."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    res = {}
    for tma in ("1", "0"):
        f = tmp_path / f"tma{tma}.npz"
        env = dict(os.environ, STKG_TMA=tma)
        subprocess.run([sys.executable, "-c", _PAD_SCRIPT, root, str(f)], check=True, env=env)
        res[tma] = dict(np.load(f))
    for k in res["1"]:
        assert np.array_equal(res["1"][k], res["0"][k]), k


_K1_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1912_10082_b200 as stk
out = {}
for ndim, n, nt in [(2, 1023, 70), (2, 45, 9), (3, 127, 5), (3, 21, 66)]:
    rng = np.random.default_rng(n + nt)
    U = torch.from_numpy(rng.standard_normal((nt, n ** ndim))).cuda()
    F = torch.from_numpy(rng.standard_normal((nt, n ** ndim))).cuda()
    p = stk.HeatPlan.p1_uniform(ndim, n, nt, transform="dense")  # K1 is backend-independent
    out[f"a{ndim}_{n}"] = p.apply(U).cpu().numpy()
    out[f"r{ndim}_{n}"] = np.array(p.residual(U, F))
np.savez(sys.argv[2], **out)
"""


def test_k1_xmarch_matches_generic(tmp_path):
    """The x-marching K1 kernels (2D and 3D; time-chunked grids, including chunk starts that
    re-derive the previous slice) against the generic kernel: operator to 1e-14, residual
    and ||F|| to 1e-12 (different summation order)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    res = {}
    for v in ("1", "0"):
        f = tmp_path / f"k1{v}.npz"
        env = dict(os.environ, STKG_K1_XMARCH=v)
        subprocess.run([sys.executable, "-c", _K1_SCRIPT, root, str(f)], check=True, env=env)
        res[v] = dict(np.load(f))
    for k in res["1"]:
        a, b = res["1"][k], res["0"][k]
        tol = 1e-14 if k.startswith("a") else 1e-12
        assert rel(a, b) < tol, (k, rel(a, b))


@pytest.mark.parametrize("ndim,n,nt", [(2, 1023, 4), (3, 127, 3), (2, 255, 40)])
def test_dst_padded_solve_deterministic(stk, cuda, ndim, n, nt):
    """Repeated solves of the padded-layout DST path (16-byte strided kernel with its shared
    tile/region reuse and per-pair named barriers, L2-prefetching contiguous kernel, scans)
    and repeated residuals are bit-identical -- a shared-memory race would show here."""
    rng = np.random.default_rng(n + nt)
    F = dev(rng.standard_normal((nt, n ** ndim)))
    p = stk.HeatPlan.p1_uniform(ndim, n, nt, transform="dst")
    U1 = host(p.solve(F))
    for _ in range(3):
        assert np.array_equal(host(p.solve(F)), U1)
    r1 = p.residual(dev(U1), F)
    assert p.residual(dev(U1), F) == r1 and r1[0] < 1e-10


@pytest.mark.parametrize("env", [{"STKG_HALF2": "20"}, {"STKG_HALF2": "21"}, {"STKG_HALF2": "41"},
                                 {"STKG_SCAN_CHUNKED": "0"}, {"STKG_SCAN_RECIP": "0"},
                                 {"STKG_FUSED": "0"}, {"STKG_FUSED_P": "2"},
                                 {"STKG_FUSED_V": "1"}, {"STKG_FUSED_V": "2"},
                                 {"STKG_FUSED_V": "3"}, {"STKG_FUSED_V": "8"},
                                 {"STKG_TRIDIAG": "0"}, {"STKG_TRI_V": "0"},
                                 {"STKG_DST_BULK": "0"}])
def test_tuning_variants_match_default(tmp_path, env):
    """The opt-in tuning variants (strided-tile shapes with and without next-tile prefetch,
    the one-chain scan for small plans, per-step division in the factored scan; the separate
    strided passes + scan instead of the fused axis-0 pass, its 2-pair tiles, carries in
    shared memory, TMA tile staging) compute the default path's solve to rounding."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    res = {}
    # the fused-DST-pass variants are compared on plans that run that pass (STKG_TRIDIAG=0:
    # uniform time grids otherwise take the line-solve pass, which ignores them)
    base = {"STKG_TRIDIAG": "0"} if any(k.startswith("STKG_FUSED") for k in env) else {}
    for tag, extra in (("v", dict(base, **env)), ("d", base)):
        f = tmp_path / f"{tag}.npz"
        subprocess.run([sys.executable, "-c", _PAD_SCRIPT, root, str(f)], check=True,
                       env=dict(os.environ, **extra))
        res[tag] = dict(np.load(f))
    # the line-solve pass and the transform-based passes are different algorithms for the same
    # solve (tridiagonal line solves vs two more sine transforms): they agree to rounding
    tol = 5e-12 if any(k.startswith("STKG_TRI") for k in env) else 1e-13
    for k in res["v"]:
        assert rel(res["v"][k], res["d"][k]) < tol, (k, rel(res["v"][k], res["d"][k]))


_FUSED_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1912_10082_b200 as stk
out = {}
for ndim, n, nt in [(2, 1023, 5), (2, 511, 4), (2, 255, 7), (2, 15, 9), (3, 127, 4), (3, 63, 3),
                    (3, 15, 6)]:
    rng = np.random.default_rng(7 * n + nt)
    F = rng.standard_normal((nt, n ** ndim))
    p = stk.HeatPlan.p1_uniform(ndim, n, nt, transform="dst")
    U = p.solve(torch.from_numpy(F).cuda())
    out[f"u{ndim}_{n}"] = U.cpu().numpy()
    out[f"r{ndim}_{n}"] = np.array(p.residual(U, torch.from_numpy(F).cuda())[0])
    # host-buffer path in 2-slice time chunks: the fused pass starts from carried modes
    pc = stk.HeatPlan.p1_uniform(ndim, n, nt, transform="dst", time_chunk=2)
    out[f"h{ndim}_{n}"] = pc.solve_host(F)
    # non-uniform temporal bidiagonals (per-step pivots)
    g = stk.SpaceGrid1D(0.0, 1.0, n)
    e = stk.p1_eigpair(g)
    M, A = stk.fem1d_matrices(g)
    D = stk.Bidiagonal(rng.uniform(1.0, 2.0, nt), rng.uniform(-1.0, -0.2, nt - 1))
    Cm = stk.Bidiagonal(rng.uniform(0.01, 0.1, nt), rng.uniform(0.01, 0.1, nt - 1))
    pn = stk.HeatPlan(stk.TensorEigPair([e] * ndim), D, Cm, [M] * ndim, [A] * ndim,
                      transform="dst", p1_h=[g.fem_h] * ndim)
    Un = pn.solve(torch.from_numpy(F).cuda())
    out[f"n{ndim}_{n}"] = Un.cpu().numpy()
    out[f"q{ndim}_{n}"] = np.array(pn.residual(Un, torch.from_numpy(F).cuda())[0])
np.savez(sys.argv[2], **out)
"""


def test_fused_axis0_pass_matches_separate_passes(tmp_path):
    """The time-marching fused axis-0 pass (heat_fused.cuh: forward DST, recurrence with the
    carries in registers, inverse DST per slice; STKG_FUSED=1 forces it for every tile
    geometry) against the separate strided passes + heat_scan_kernel (STKG_FUSED=0): device
    solves, host-buffer solves in 2-slice chunks (carried modes, l0 > 0) and non-uniform
    temporal bidiagonals, 2D and 3D, N = 16 ... 1024.  Agreement to 1e-12 (the fused pass
    multiplies by a Newton reciprocal where the scan divides); GPU residuals <= 1e-11."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    res = {}
    for v in ("1", "0"):
        f = tmp_path / f"fused{v}.npz"
        subprocess.run([sys.executable, "-c", _FUSED_SCRIPT, root, str(f)], check=True,
                       env=dict(os.environ, STKG_FUSED=v, STKG_TRIDIAG="0"))
        res[v] = dict(np.load(f))
    for k in res["1"]:
        a, b = res["1"][k], res["0"][k]
        if k[0] in "rq":
            assert float(a) < 1e-11, (k, float(a))
        else:
            assert rel(a, b) < 1e-12, (k, rel(a, b))
    for k in res["1"]:
        if k[0] == "h":
            assert rel(res["1"][k], res["1"]["u" + k[1:]]) < 1e-13, k


_LINE_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1912_10082_b200 as stk
out = {}
for ndim, n, nt in [(2, 1023, 5), (2, 511, 4), (2, 255, 7), (2, 127, 6), (2, 63, 5), (3, 127, 4),
                    (3, 63, 3)]:
    rng = np.random.default_rng(7 * n + nt)
    F = rng.standard_normal((nt, n ** ndim))
    T = nt / (n + 1.0)  # dt = h: a time step in proportion to the mesh, as in the configs
    p = stk.HeatPlan.p1_uniform(ndim, n, nt, T=T, transform="dst")
    out[f"s{ndim}_{n}"] = np.array(["separate", "fused_dst", "line_solve"].index(p.schedule()))
    Fd = torch.from_numpy(F).cuda()
    U = p.solve(Fd)
    out[f"u{ndim}_{n}"] = U.cpu().numpy()
    out[f"r{ndim}_{n}"] = np.array(p.residual(U, Fd)[0])
    # host-buffer path in 2-slice time chunks: every launch starts from the carried z_{l0-1}
    pc = stk.HeatPlan.p1_uniform(ndim, n, nt, T=T, transform="dst", time_chunk=2)
    out[f"h{ndim}_{n}"] = pc.solve_host(F)
# a longer time axis on a domain / horizon that is not the unit one (other stencil scales)
p = stk.HeatPlan.p1_uniform(2, 255, 96, T=10.0, a=-1.0, b=1.0, transform="dst")
F = np.random.default_rng(5).standard_normal((96, 255 * 255))
Fd = torch.from_numpy(F).cuda()
U = p.solve(Fd)
out["s_long"] = np.array(["separate", "fused_dst", "line_solve"].index(p.schedule()))
out["u_long"] = U.cpu().numpy()
out["r_long"] = np.array(p.residual(U, Fd)[0])
# non-uniform temporal bidiagonals: the TMA variant recomputes its per-column constants every
# step; the LDL^T variant (per-plan pivot table) leaves them to the transform-based pass
for ndim, n, nt in [(2, 1023, 6), (2, 255, 9), (3, 127, 5)]:
    rng = np.random.default_rng(11 + n)
    g = stk.SpaceGrid1D(0.0, 1.0, n)
    e = stk.p1_eigpair(g)
    M, A = stk.fem1d_matrices(g)
    D = stk.Bidiagonal(rng.uniform(1.0, 2.0, nt), rng.uniform(-1.0, -0.2, nt - 1))
    cscale = 16.0 / (n + 1)  # time steps in proportion to the mesh
    Cm = stk.Bidiagonal(cscale * rng.uniform(0.01, 0.1, nt), cscale * rng.uniform(0.01, 0.1, nt - 1))
    F = rng.standard_normal((nt, n ** ndim))
    Fd = torch.from_numpy(F).cuda()
    pn = stk.HeatPlan(stk.TensorEigPair([e] * ndim), D, Cm, [M] * ndim, [A] * ndim,
                      transform="dst", p1_h=[g.fem_h] * ndim)
    out[f"S{ndim}_{n}"] = np.array(["separate", "fused_dst", "line_solve"].index(pn.schedule()))
    Un = pn.solve(Fd)
    out[f"n{ndim}_{n}"] = Un.cpu().numpy()
    out[f"q{ndim}_{n}"] = np.array(pn.residual(Un, Fd)[0])
    pc = stk.HeatPlan(stk.TensorEigPair([e] * ndim), D, Cm, [M] * ndim, [A] * ndim,
                      transform="dst", p1_h=[g.fem_h] * ndim, time_chunk=2)
    out[f"c{ndim}_{n}"] = pc.solve_host(F)
np.savez(sys.argv[2], **out)
"""


def test_line_solve_pass_matches_transform_passes(tmp_path):
    """The time-marching line-solve axis-0 pass (heat_tridiag.cuh: axis 0 is not transformed;
    per column and slice one Toeplitz tridiagonal solve by constant-coefficient causal /
    anti-causal sweeps, TMA tile loads and stores; STKG_FUSED=1 forces the time-marching
    schedule for every tile geometry) against the transform-based schedule (STKG_TRIDIAG=0)
    and against the cp.async LDL^T variant of the same pass (STKG_TRI_V=0): device solves,
    host-buffer solves in 2-slice chunks (carried state, l0 > 0), 2D and 3D, N = 64 ... 1024,
    a non-unit domain and horizon; non-uniform time grids (per-step constants in the TMA
    variant, the transform pass under the LDL^T variant).  Agreement to 5e-12 (different
    algorithms for the same solve), GPU residuals <= 1e-11."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    res = {}
    for tag, env in (("line", {}), ("dst", {"STKG_TRIDIAG": "0"}), ("ldl", {"STKG_TRI_V": "0"})):
        f = tmp_path / f"{tag}.npz"
        subprocess.run([sys.executable, "-c", _LINE_SCRIPT, root, str(f)], check=True,
                       env=dict(os.environ, STKG_FUSED="1", **env))
        res[tag] = dict(np.load(f))
    for k, a in res["line"].items():
        if k[0] == "s":  # uniform grids: both line-solve variants
            assert int(a) == 2 and int(res["ldl"][k]) == 2 and int(res["dst"][k]) == 1, k
        elif k[0] == "S":  # non-uniform grids: the TMA variant only
            assert int(a) == 2 and int(res["ldl"][k]) == 1 and int(res["dst"][k]) == 1, k
        elif k[0] in "rq":
            assert float(a) < 1e-11 and float(res["ldl"][k]) < 1e-11, (k, float(a))
        else:
            assert rel(a, res["dst"][k]) < 5e-12, (k, rel(a, res["dst"][k]))
            assert rel(res["ldl"][k], res["dst"][k]) < 5e-12, (k, rel(res["ldl"][k], res["dst"][k]))
    for k in res["line"]:
        if k[0] == "h":
            assert rel(res["line"][k], res["line"]["u" + k[1:]]) < 1e-13, k
        if k[0] == "c":
            assert rel(res["line"][k], res["line"]["n" + k[1:]]) < 1e-13, k


def test_line_solve_conditioning_gate(stk, cuda):
    """A tridiagonal line solve loses cond(T_c) ulps, the modal recurrence none: plans whose
    time step is very large against h^2 (cond > 1e5) keep the transform pass, and both
    schedules stay within 2e-12 of the dense DMMA backend."""
    n, nt = 1023, 2
    F = np.random.default_rng(5).standard_normal((nt, n * n))
    for T, want in ((1.0, "fused_dst"), (nt / 1024.0, "line_solve")):
        pd = stk.HeatPlan.p1_uniform(2, n, nt, T=T, transform="dense")
        ps = stk.HeatPlan.p1_uniform(2, n, nt, T=T, transform="dst")
        assert ps.schedule() == want, (T, ps.schedule())
        Ud, Us = host(pd.solve(dev(F))), host(ps.solve(dev(F)))
        assert rel(Us, Ud) < 2e-12, (T, rel(Us, Ud))


_OVERLAP_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1912_10082_b200 as stk
out = {}
for n, nt in [(1023, 40), (1023, 37), (511, 64)]:
    F = np.random.default_rng(n + nt).standard_normal((nt, n * n))
    p = stk.HeatPlan.p1_uniform(2, n, nt, transform="dst")
    Fd = torch.from_numpy(F).cuda()
    U = p.solve(Fd)
    out[f"u{n}_{nt}"] = U.cpu().numpy()
    U2 = p.solve(Fd)  # repeated: tickets and events reused
    out[f"v{n}_{nt}"] = U2.cpu().numpy()
    out[f"r{n}_{nt}"] = np.array(p.residual(U, Fd)[0])
# host-buffer path in 40-slice chunks: the overlapped schedule with carried modes (l0 > 0)
F = np.random.default_rng(3).standard_normal((80, 1023 * 1023))
ph = stk.HeatPlan.p1_uniform(2, 1023, 80, transform="dst", time_chunk=40)
out["h1023_80"] = ph.solve_host(F)
np.savez(sys.argv[2], **out)
"""


@pytest.mark.parametrize("k", ["4", "3"])
def test_overlapped_schedule_bit_identical(tmp_path, k):
    """The overlapped 2D schedule (time chunks; contiguous passes with ticketed items on a
    low-priority stream beside the fused pass on a high-priority stream, carries across
    chunks) computes exactly what the sequential passes compute: same arithmetic per slice,
    only the launch order differs.  Uneven chunks (n_t = 37), repeated solves.  (Plans that
    take the line-solve pass keep the plain order; STKG_TRIDIAG=0 selects the fused DST pass,
    the schedule of non-uniform time grids.)"""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    res = {}
    for v in (k, "0"):
        f = tmp_path / f"ov{v}.npz"
        subprocess.run([sys.executable, "-c", _OVERLAP_SCRIPT, root, str(f)], check=True,
                       env=dict(os.environ, STKG_OVERLAP=v, STKG_TRIDIAG="0"))
        res[v] = dict(np.load(f))
    for key in res["0"]:
        a, b = res[k][key], res["0"][key]
        assert np.array_equal(a, b), (key, float(np.abs(a - b).max()),
                                      np.argwhere(a != b)[:4].tolist() if a.ndim else None)
        if key[0] == "r":
            assert float(res[k][key]) < 1e-11
