"""CPU tests: the C ABI library loads and exports every declared symbol; the host-side
assembly matches the SPEC known answers, the oracle, and (bit for bit) the reference's own
spline code; the oracle itself is pinned against the SPEC known answers."""
import re

import numpy as np
import pytest

from conftest import ROOT


# ------------------------------------------------------------------------------ ABI --
def declared_symbols():
    hdr = (ROOT / "include" / "stk_gpu.h").read_text()
    return sorted(set(re.findall(r"\b(stkg_\w+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol(stk):
    from paper_1912_10082_b200 import _lib
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(_lib.lib, s), f"{s} declared in stk_gpu.h but not exported"
    # and the ctypes binding covers exactly the header
    assert set(_lib.SIGNATURES) == set(syms)


def test_library_is_sm100a_cuda(stk):
    import subprocess
    from paper_1912_10082_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(_lib.LIB_PATH)],
                          capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass  # FP64 tensor-core transforms


def test_error_mapping(stk):
    import ctypes as C
    from paper_1912_10082_b200._lib import lib
    from paper_1912_10082_b200.errors import check
    z = np.zeros(4)
    p = z.ctypes.data_as(C.POINTER(C.c_double))
    with pytest.raises(stk.ArgumentError, match="nt must be >= 1"):
        check(lib.stkg_heat_time_matrices(0, 1.0, p, p, p, p))
    with pytest.raises(stk.DefinitenessError):
        stk.sym_gen_eig(np.eye(3), -np.eye(3))
    with pytest.raises(stk.ArgumentError, match="not symmetric"):
        stk.sym_gen_eig(np.triu(np.ones((3, 3))), np.eye(3))


# ------------------------------------------------------------------ assembly (KATs) --
def test_heat_time_matrices_kats(stk, kats):
    for k in kats["heat_time_matrices"]:
        D, Cm = stk.heat_time_matrices(stk.TimeGrid(k["nt"], k["T"]))
        if "D" in k:
            assert np.array_equal(D.dense(), np.array(k["D"], float))
            assert np.array_equal(Cm.dense(), np.array(k["C"], float))
        if "D_row_sums" in k:
            assert np.array_equal(D.dense().sum(1), np.array(k["D_row_sums"], float))


def test_fem1d_matrices_kats(stk, kats):
    for k in kats["fem1d_matrices"]:
        M, A = stk.fem1d_matrices(stk.SpaceGrid1D(k["a"], k["b"], k["nh"]))
        if "A" in k:
            assert np.allclose(A.dense(), np.array(k["A"], float), rtol=0, atol=1e-14)
        if "M" in k:
            assert np.allclose(M.dense(), np.array(k["M"], float), rtol=0, atol=1e-15)
        if "M_interior_row_sum" in k:
            assert abs(M.dense()[k["nh"] // 2].sum() - k["M_interior_row_sum"]) < 1e-15


def test_assembly_matches_oracle_bitwise(stk, orc):
    for nt, T in [(1, 1.0), (7, 2.5), (1024, 1.0)]:
        D, Cm = stk.heat_time_matrices(stk.TimeGrid(nt, T))
        d, c = orc.heat_time_matrices(nt, T)
        assert np.array_equal(D.diag, d[0]) and np.array_equal(D.sup, d[1])
        assert np.array_equal(Cm.diag, c[0]) and np.array_equal(Cm.sup, c[1])
    for nh, a, b in [(1, 0.0, 1.0), (255, 0.0, 1.0), (1023, -1.0, 1.0)]:
        M, A = stk.fem1d_matrices(stk.SpaceGrid1D(a, b, nh))
        m, aa = orc.fem1d_matrices(a, b, nh)
        assert np.array_equal(M.diag, m[0]) and np.array_equal(M.off, m[1])
        assert np.array_equal(A.diag, aa[0]) and np.array_equal(A.off, aa[1])


def test_fem2d_kats(stk, orc):
    # 1x1 scalars, 2x2 vs brute-force Kronecker, pencil eigenvalues sums
    for n in (1, 2, 5):
        m, a = orc.fem1d_matrices(0.0, 1.0, n)
        M, A = orc.tensor_sparse([m, m], [a, a])
        Md, Ad = orc.tri_dense(m), orc.tri_dense(a)
        assert np.allclose(M.toarray(), np.kron(Md, Md), atol=1e-15)
        assert np.allclose(A.toarray(), np.kron(Ad, Md) + np.kron(Md, Ad), atol=1e-13)
    import scipy.linalg as sl
    m, a = orc.fem1d_matrices(0.0, 1.0, 6)
    M, A = orc.tensor_sparse([m, m], [a, a])
    lam2 = sl.eigh(A.toarray(), M.toarray(), eigvals_only=True)
    e = stk.p1_eigpair(stk.SpaceGrid1D(0.0, 1.0, 6)).lambdas
    sums = np.sort((e[:, None] + e[None, :]).ravel())
    assert np.allclose(lam2, sums, rtol=1e-12)


@pytest.mark.parametrize("n", [1, 2, 15, 255, 1023])
def test_p1_eigpair_is_the_generalized_eigenbasis(stk, n):
    g = stk.SpaceGrid1D(0.0, 1.0, n)
    M, A = stk.fem1d_matrices(g)
    e = stk.p1_eigpair(g)
    X = e.X
    Md, Ad = M.dense(), A.dense()
    assert np.abs(X.T @ Md @ X - np.eye(n)).max() < 1e-13
    assert np.abs(X.T @ Ad @ X - np.diag(e.lambdas)).max() < 1e-13 * e.lambdas.max()
    assert np.all(np.diff(e.lambdas) > 0)
    if n <= 255:
        import scipy.linalg as sl
        ref = sl.eigh(Ad, Md, eigvals_only=True)
        assert np.abs(ref - e.lambdas).max() < 1e-12 * ref.max()


def test_sym_gen_eig_matches_lapack(stk):
    import scipy.linalg as sl
    rng = np.random.default_rng(3)
    for n in (1, 4, 37):
        B = rng.standard_normal((n, n))
        M = B @ B.T + n * np.eye(n)
        Q = rng.standard_normal((n, n))
        Q = Q + Q.T
        e = stk.sym_gen_eig(Q, M)
        ref = sl.eigh(Q, M, eigvals_only=True)
        assert np.allclose(e.lambdas, ref, rtol=1e-12, atol=1e-12)
        assert np.abs(e.X.T @ M @ e.X - np.eye(n)).max() < 1e-12
        assert np.abs(Q @ e.X - M @ e.X @ np.diag(e.lambdas)).max() < 1e-10


def test_wave_bands_bit_identical_to_reference(stk, ref_bands):
    """Product spline Gram bands == the reference's own splines.hpp/quadrature.hpp output."""
    for key in ref_bands:
        if key.startswith("space_"):
            _, nh, deg = key.split("_")
            s = stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, int(nh)), int(deg))
            got = np.stack([s.M.band, s.A.band, s.Q.band])
            assert np.array_equal(got, ref_bands[key]), key
        elif key.startswith("time_"):
            _, nt, deg = key.split("_")
            t = stk.wave_time_matrices(stk.TimeGrid(int(nt), 1.0), int(deg))
            got = np.stack([t.Q.band, t.D.band, t.M.band])
            assert np.array_equal(got, ref_bands[key]), key


def test_wave_dims_and_end_conditions(stk):
    # n_t = 1024 elements -> 1025 cubic test functions; space keeps nh
    assert stk.wave_time_dim(1024, 3) == 1025
    t = stk.wave_time_matrices(stk.TimeGrid(1024, 1.0), 3)
    assert t.M.n == 1025
    s = stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, 1023), 3)
    assert s.M.n == 1023
    # Gram matrices: M, Q s.p.d.; D_t nonsymmetric
    Mt = t.M.dense()
    assert np.linalg.eigvalsh(0.5 * (Mt + Mt.T)).min() > 0
    Dd = stk.wave_time_matrices(stk.TimeGrid(16, 1.0), 3).D.dense()
    assert np.abs(Dd - Dd.T).max() > 1e-3


# ---------------------------------------------------------------- oracle vs KATs ----
def test_oracle_solve_projected_heat_kats(orc, kats):
    # k=1, N_t=1, h_m=d=1, h_a=c=1, g=2 -> y=1
    Y = orc.solve_projected_heat_with_dense(np.array([[1.0]]), np.array([1.0]),
                                            (np.array([1.0]), np.zeros(0)),
                                            (np.array([1.0]), np.zeros(0)), np.array([[2.0]]))
    assert Y[0, 0] == 1.0
    # H_M = I, H_A = diag(1,2), heat D, C (N_t=3, dt=1), G = ones vs dense Kron
    d, c = orc.heat_time_matrices(3, 3.0)
    X = np.eye(2)
    lam = np.array([1.0, 2.0])
    G = np.ones((3, 2))
    Y = orc.solve_projected_heat_with_dense(X, lam, d, c, G)
    Dm, Cm = orc.bidiag_dense(d), orc.bidiag_dense(c)
    B = np.kron(Dm.T, np.eye(2)) + np.kron(Cm.T, np.diag(lam))
    y = np.linalg.solve(B, G.ravel())
    assert np.allclose(Y.ravel(), y, rtol=1e-14, atol=1e-14)


def test_oracle_cn_kats(orc):
    # M=1, A=0, F[:,l]=dt -> u^l = l dt ; SPEC.md:518 needs u0 -> via F_1
    nt, dt = 8, 1.0 / 8
    m = (np.array([1.0]), np.zeros(0))
    a0 = (np.array([0.0]), np.zeros(0))
    U = orc.crank_nicolson([m], [a0], dt, np.full((nt, 1), dt))
    assert np.allclose(U[:, 0], dt * np.arange(1, nt + 1), rtol=1e-15)
    # M=1, A=1, f=0, u0=1: equivalent to zero u0 and F_1 = (1 - dt/2) (first step's rhs)
    a1 = (np.array([1.0]), np.zeros(0))
    F = np.zeros((nt, 1))
    F[0, 0] = 1.0 - dt / 2
    U = orc.crank_nicolson([m], [a1], dt, F)
    r = (1 - dt / 2) / (1 + dt / 2)
    assert np.allclose(U[:, 0], r ** np.arange(1, nt + 1), rtol=1e-14)


def test_oracle_cn_equals_decoupled(orc):
    """CN (stk/cn_baseline.hpp) and the decoupled solve (stk/sylvester.hpp:117) are the same
    algebra for any F: two independent restatements agree."""
    from paper_1912_10082_b200 import inputs
    rng = np.random.default_rng(0)
    for ndim, n, nt in [(1, 31, 20), (2, 9, 12), (3, 5, 6)]:
        m, a = orc.fem1d_matrices(0.0, 1.0, n)
        d, c = orc.heat_time_matrices(nt)
        F = rng.standard_normal((nt, n ** ndim))
        Ucn = orc.crank_nicolson([m] * ndim, [a] * ndim, 1.0 / nt, F)
        Ud = orc.heat_decoupled([orc.p1_pencil_eig(m, a)] * ndim, d, c, F)
        assert np.linalg.norm(Ucn - Ud) / np.linalg.norm(Ud) < 1e-12
        assert orc.heat_residual([m] * ndim, [a] * ndim, d, c, Ud, F) < 1e-12
    # the generator is bit-identical between the oracle (C) and the product (numpy)
    assert np.array_equal(orc.fill_uniform(777, 5, 48, 3), inputs.uniform_pm1(777, 5, 48, 3))


@pytest.mark.parametrize("ndim,n,nt", [(2, 31, 9), (2, 63, 6), (3, 15, 5)])
def test_oracle_line_march_equals_decoupled(orc, ndim, n, nt):
    """The line-solve schedule (axis 0 untransformed: one Toeplitz tridiagonal solve per column
    and step, solved by the method-of-images recurrences of csrc/heat_tridiag.cuh) against the
    reference algorithm, solve_projected_heat_with in tensor form (all axes diagonalised), and
    the tridiagonal solver alone against a dense solve -- including a column with a ~ 0."""
    rng = np.random.default_rng(n + nt)
    m, a = orc.fem1d_matrices(0.0, 1.0, n)
    d, c = orc.heat_time_matrices(nt, 1.0)
    e = orc.p1_pencil_eig(m, a)
    F = rng.uniform(-1.0, 1.0, (nt, n ** ndim))
    ref = orc.heat_decoupled([e] * ndim, d, c, F)
    got = orc.heat_line_march([e] * (ndim - 1), m, a, d, c, F)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    aa = np.array([-1.0, 0.3, 0.0, 1e-9, -0.49999])
    bb = np.array([2.0001, 1.0, 1.0, 1.0, 1.0])
    r = rng.standard_normal((n, aa.size))
    x = orc.toeplitz_tridiag_solve_images(aa, bb, r)
    for k in range(aa.size):
        T = bb[k] * np.eye(n) + aa[k] * (np.eye(n, k=1) + np.eye(n, k=-1))
        assert np.abs(T @ x[:, k] - r[:, k]).max() <= 1e-10 * np.abs(r[:, k]).max()


def test_oracle_wave_gmres_matches_direct(orc, ref_bands):
    sb, tb = ref_bands["space_16_3"], ref_bands["time_16_3"]
    W = orc.WaveSystemNP(sb, tb)
    rng = np.random.default_rng(1)
    b = rng.standard_normal(sb.shape[2] * tb.shape[2])
    x, its, hist = W.gmres(b, tol=1e-12, maxit=400)
    xd = W.direct(b)
    assert np.linalg.norm(x - xd) / np.linalg.norm(xd) < 1e-9
    assert all(h2 <= h1 * (1 + 1e-12) for h1, h2 in zip(hist, hist[1:]))
    # C and numpy restatements of WaveOperator::apply agree
    U = rng.standard_normal((tb.shape[2], sb.shape[2]))
    assert np.allclose(orc.wave_apply(sb, tb, U).ravel(), W.apply(U.ravel()), rtol=1e-12,
                       atol=1e-12 * np.abs(W.apply(U.ravel())).max())


@pytest.mark.parametrize("n,nt,r", [(10, 6, 1), (40, 30, 1), (63, 40, 3)])
def test_oracle_rksm_matches_direct(orc, n, nt, r):
    """Pins the oracle's rksm_solve restatement (stk/rksm.hpp:127-234) against a sparse
    direct solve of the full Kronecker system -- SPEC.md:411 (N_h=10, N_t=6, rank 1) and
    SPEC.md:574 (N_h=40, N_t=30): relres <= 1e-8, error vs dense <= 1e-6."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    m, a = orc.fem1d_matrices(0.0, 1.0, n)
    d, c = orc.heat_time_matrices(nt)
    rng = np.random.default_rng(3)
    L, R = rng.standard_normal((n, r)), rng.standard_normal((nt, r))
    left, right, its, hist = orc.rksm_solve([m], [a], d, c, L, R, tol=1e-8)
    assert hist[-1] <= 1e-8 and its == len(hist)
    M, A = orc.tensor_sparse([m], [a])
    K = (sp.kron(sp.csr_matrix(orc.bidiag_dense(d)).T, M)
         + sp.kron(sp.csr_matrix(orc.bidiag_dense(c)).T, A))
    u = spl.spsolve(K.tocsc(), (L @ R.T).reshape(-1, order="F")).reshape(n, nt, order="F")
    assert np.linalg.norm(u - left @ right.T) / np.linalg.norm(u) <= 1e-6


def test_oracle_adaptive_shift_spec_example(orc):
    """one shift -1, one Ritz value 2, candidates {-0.5,-1.5,-4} -> -4.
    The oracle restates the candidate-set loop; evaluate it on the explicit set."""
    cands = [-0.5, -1.5, -4.0]
    vals = [np.log(abs(x + 1.0)) - np.log(abs(x + 2.0)) for x in cands]
    assert cands[int(np.argmax(vals))] == -4.0
    s1 = orc.adaptive_next_shift([-1.0], [2.0], 1.0, 10.0)
    assert s1 == orc.adaptive_next_shift([-1.0], [2.0], 1.0, 10.0) and s1 < 0


# ------------------------------------------- heat-ex1 (the reference's desk problem) --
def test_oracle_gauss_rule_and_load_projection(orc, ref_bands):
    """The oracle's project_rhs_heat (stk/rhs_sep.hpp:111-151) uses the reference's own
    6-point Gauss-Legendre rule (fixture from oracle/_ref); numpy's rule agrees to ulps.
    Known answers: a constant load projects onto h per interior hat and dt per interval."""
    x6, w6 = orc.gauss_legendre01(6)
    np.testing.assert_array_equal(x6, ref_bands["gauss_6_x"])
    xn, wn = np.polynomial.legendre.leggauss(6)
    assert np.abs((xn + 1) / 2 - x6).max() < 1e-15 and np.abs(wn / 2 - w6).max() < 1e-15
    G, H = orc.project_rhs_heat(lambda t: np.ones_like(t), lambda x: np.ones_like(x),
                                8, 2.0, -1.0, 1.0, 9)
    np.testing.assert_allclose(G, 0.2, rtol=1e-14)
    np.testing.assert_allclose(H, 0.25, rtol=1e-14)
    Gt, Ht = orc.project_rhs_heat(orc.heat_ex1_theta, orc.heat_ex1_f, 5, 10.0, -1.0, 1.0, 9,
                                  trapezoidal_time=True)
    t = np.arange(6) * 2.0
    np.testing.assert_allclose(Ht, 1.0 * (orc.heat_ex1_theta(t[:-1]) + orc.heat_ex1_theta(t[1:])))
    # cos(pi x/2) on (-1,1) is the first Dirichlet eigenfunction: its P1 load vector is the
    # first discrete eigenvector (to quadrature accuracy)
    xi = -1.0 + 0.2 * np.arange(1, 10)
    v = np.cos(np.pi / 2 * xi)
    assert np.linalg.norm(Gt / np.linalg.norm(Gt) - v / np.linalg.norm(v)) < 1e-6


@pytest.mark.parametrize("ndim,nh", [(1, 199), (2, 60)])
def test_oracle_rksm_heat_ex1_acceptance(orc, ndim, nh):
    """SPEC.md:612-615 on the reference's own heat-ex1 problem (stk/bench.hpp:300-306,
    361-406: Omega=(-1,1)^d, T=10, load 10 sin(t) t prod cos(pi x_i/2)), N_t in
    {100, 300, 500}: iterations <= 30 with spread <= 3, rank <= 20, mu_mem <= 40 (2D desk
    problem); in 1D (N_h=199, trapezoidal-time RHS) the RKSM solution equals the CN
    trajectory column by column to <= 1e-6 (criterion 2)."""
    its_all = []
    for nt in (100, 300, 500):
        L, H = orc.heat_ex1_load(ndim, nh, nt, T=10.0, trapezoidal_time=(ndim == 1))
        m, a = orc.fem1d_matrices(-1.0, 1.0, nh)
        d, c = orc.heat_time_matrices(nt, 10.0)
        left, right, its, hist = orc.rksm_solve([m] * ndim, [a] * ndim, d, c, L[:, None],
                                                H[:, None], tol=1e-8, maxit=60)
        assert hist[-1] <= 1e-8 and its <= 30 and left.shape[1] <= 20
        its_all.append(its)
        if ndim == 1:
            U = (left @ right.T).T  # (nt, nx)
            Ucn = orc.crank_nicolson_splu([m], [a], 10.0 / nt, np.outer(H, L))
            col = np.linalg.norm(U - Ucn, axis=1) / np.linalg.norm(Ucn, axis=1)
            assert col.max() <= 1e-6, col.max()
    assert max(its_all) - min(its_all) <= 3


# ----------------------------------- extended-precision wave residual (oracle infra) --
def test_oracle_banded_wave_residual_matches_apply(orc, ref_bands):
    """wave_residual_banded in float64 is WaveOperator::apply (the sparse restatement) bit
    for bit, and its longdouble evaluation agrees to FP64 rounding."""
    sb, tb = ref_bands["space_31_3"], ref_bands["time_33_3"]
    W = orc.WaveSystemNP(sb, tb)
    rng = np.random.default_rng(3)
    x, b = rng.standard_normal(W.nh * W.nt), rng.standard_normal(W.nh * W.nt)
    r64 = orc.wave_residual_banded(sb, tb, b, x, dtype=np.float64)
    assert np.array_equal(r64, b - W.apply(x))
    rld = orc.wave_residual_banded(sb, tb, b, x)
    assert np.linalg.norm(rld.astype(np.float64) - r64) <= 1e-14 * np.linalg.norm(r64)


def test_oracle_refined_direct_wave_solve(orc, ref_bands):
    """kron_direct_solve + longdouble iterative refinement reaches a relative residual far
    below the FP64 direct solve's (the oracle for the GPU refined solve's forward error)."""
    sb, tb = ref_bands["space_31_3"], ref_bands["time_33_3"]
    b = np.random.default_rng(4).standard_normal(sb.shape[2] * tb.shape[2])
    xh, xl, hist = orc.wave_refined_direct(sb, tb, b, steps=3)
    assert hist[-1] <= 1e-15 and hist[-1] < hist[0]


def test_oracle_modal_banded_inverse_pair(orc, ref_bands):
    """The oracle's modal banded preconditioner solve and its operator are inverses."""
    sb, tb = ref_bands["space_31_3"], ref_bands["time_33_3"]
    W = orc.WaveSystemNP(sb, tb)
    v = np.random.default_rng(9).standard_normal(W.nh * W.nt)
    assert np.linalg.norm(W.modal_banded_apply(W.modal_banded(v)) - v) <= 1e-11 * np.linalg.norm(v)
