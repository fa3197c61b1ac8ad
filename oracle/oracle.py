"""CPU oracle for the B200 Kronecker space-time solver -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs
may import this module; the product package never does.  Two independent restatements of
the reference algorithms live here:

* ``C`` -- ``libstk_oracle.so`` (stk_oracle.c): loop-for-loop restatements of
  heat_time_matrices / fem1d_matrices (stk/discretize.hpp:44-77), KronOp::apply
  (stk/sylvester.hpp:32-38), solve_projected_heat_with (:117-142), crank_nicolson
  (stk/cn_baseline.hpp:26-48, banded Cholesky in place of SimplicialLLT) and
  WaveOperator::apply (stk/outer_krylov.hpp:178-186);
* numpy/scipy -- tensor-form decoupled heat solve with scipy ``eigh`` eigenbases (not the
  closed form the product uses), CN with ``scipy.sparse.linalg.splu``, TwoTermPrecond::solve
  (stk/sylvester.hpp:168-176), and gmres (stk/outer_krylov.hpp:75-164, modified Gram-Schmidt
  + one re-orthogonalisation pass, exactly as the reference).

``ref`` -- ``oracle/_ref/libstkref.so`` is the reference's own splines.hpp/quadrature.hpp
compiled from /root/reference (only in the build container); tests/golden holds the band
fixtures it produced so the GPU box can check them without the reference tree.

Parity status: the heat path is pinned by the SPEC.md known-answer examples
(tests/golden/spec_kats.json) and by oracle-vs-oracle agreement (CN vs decoupled); the wave
assembly is pinned bit-for-bit by the reference's own spline code.  No reference-produced
golden vectors exist for the solver outputs (the reference cannot be built: no Eigen3).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_dp = C.POINTER(C.c_double)


def _build_c():
    so = HERE / "libstk_oracle.so"
    src = HERE / "stk_oracle.c"
    if not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE), "libstk_oracle.so"], check=True,
                       capture_output=True)
    return so


def _lib():
    lib = C.CDLL(str(_build_c()))
    i64p = C.POINTER(C.c_int64)
    pp = C.POINTER(_dp)
    lib.or_heat_apply.argtypes = [C.c_int, i64p, C.c_int64, pp, pp, pp, pp, _dp, _dp, _dp, _dp,
                                  _dp, _dp]
    lib.or_solve_projected_heat_with.argtypes = [C.c_int64, C.c_int64, _dp, _dp, _dp, _dp, _dp,
                                                 _dp, _dp, _dp]
    lib.or_solve_projected_heat_with.restype = C.c_int
    lib.or_crank_nicolson.argtypes = [C.c_int, i64p, C.c_int64, C.c_double, pp, pp, pp, pp,
                                      _dp, _dp]
    lib.or_crank_nicolson.restype = C.c_int
    lib.or_wave_apply.argtypes = [C.c_int64, C.c_int64, _dp, _dp, _dp, _dp]
    lib.or_fill_uniform.argtypes = [_dp, C.c_int64, C.c_uint64, C.c_uint64, C.c_int64]
    lib.or_heat_time_matrices.argtypes = [C.c_int, C.c_double, _dp, _dp, _dp, _dp]
    lib.or_fem1d_matrices.argtypes = [C.c_double, C.c_double, C.c_int, _dp, _dp, _dp, _dp]
    return lib


clib = _lib()


def _p(a):
    return a.ctypes.data_as(_dp)


def _arr_pp(arrs, keep):
    out = (_dp * 3)()
    for i, a in enumerate(arrs):
        a = np.ascontiguousarray(a, dtype=np.float64)
        if a.size == 0:
            a = np.zeros(1)
        keep.append(a)
        out[i] = _p(a)
    return out


# ------------------------------------------------------------------------ assembly --
def heat_time_matrices(nt: int, T: float = 1.0):
    dd, cd = np.empty(nt), np.empty(nt)
    ds, cs = np.zeros(max(nt - 1, 1)), np.zeros(max(nt - 1, 1))
    clib.or_heat_time_matrices(nt, T, _p(dd), _p(ds), _p(cd), _p(cs))
    return (dd, ds[: nt - 1]), (cd, cs[: nt - 1])


def fem1d_matrices(a: float, b: float, nh: int):
    md, ad = np.empty(nh), np.empty(nh)
    mo, ao = np.zeros(max(nh - 1, 1)), np.zeros(max(nh - 1, 1))
    clib.or_fem1d_matrices(a, b, nh, _p(md), _p(mo), _p(ad), _p(ao))
    return (md, mo[: nh - 1]), (ad, ao[: nh - 1])


def tri_dense(t):
    d, o = t
    m = np.diag(d)
    if d.size > 1:
        m = m + np.diag(o, 1) + np.diag(o, -1)
    return m


def bidiag_dense(b):
    d, s = b
    m = np.diag(d)
    if d.size > 1:
        m = m + np.diag(s, 1)
    return m


def tensor_sparse(ms, as_):
    """fem2d_matrices (stk/discretize.hpp:81-88) / 3D restatement as scipy CSR."""
    import scipy.sparse as sp
    M1 = [sp.csr_matrix(tri_dense(m)) for m in ms]
    A1 = [sp.csr_matrix(tri_dense(a)) for a in as_]
    M = M1[0]
    for m in M1[1:]:
        M = sp.kron(M, m, format="csr")
    A = None
    for k in range(len(ms)):
        t = A1[0] if k == 0 else M1[0]
        for j in range(1, len(ms)):
            t = sp.kron(t, A1[j] if j == k else M1[j], format="csr")
        A = t if A is None else A + t
    return M.tocsr(), A.tocsr()


# ------------------------------------------------------------------------ heat (C) --
def heat_apply(ms, as_, d, c, U):
    """C restatement of KronOp::apply (stk/sylvester.hpp:32-38); U is (nt, nx) C-order."""
    ndim = len(ms)
    n = (C.c_int64 * 3)(*[m[0].size for m in ms], *([1] * (3 - ndim)))
    keep = []
    U = np.ascontiguousarray(U, dtype=np.float64)
    out = np.empty_like(U)
    clib.or_heat_apply(ndim, n, U.shape[0], _arr_pp([m[0] for m in ms], keep),
                       _arr_pp([m[1] for m in ms], keep), _arr_pp([a[0] for a in as_], keep),
                       _arr_pp([a[1] for a in as_], keep), _p(np.ascontiguousarray(d[0])),
                       _p(np.ascontiguousarray(d[1]) if d[1].size else np.zeros(1)),
                       _p(np.ascontiguousarray(c[0])),
                       _p(np.ascontiguousarray(c[1]) if c[1].size else np.zeros(1)), _p(U),
                       _p(out))
    return out


def solve_projected_heat_with_dense(X, lam, d, c, G):
    """C restatement of solve_projected_heat_with with a dense k x k EigPair."""
    k = X.shape[0]
    G = np.ascontiguousarray(G, dtype=np.float64)
    nt = G.shape[0]
    Xc = np.asfortranarray(X)
    Y = np.empty_like(G)
    dsup = d[1] if d[1].size else np.zeros(1)
    csup = c[1] if c[1].size else np.zeros(1)
    st = clib.or_solve_projected_heat_with(k, nt, _p(Xc), _p(np.ascontiguousarray(lam)),
                                           _p(np.ascontiguousarray(d[0])), _p(np.ascontiguousarray(dsup)),
                                           _p(np.ascontiguousarray(c[0])), _p(np.ascontiguousarray(csup)),
                                           _p(G), _p(Y))
    if st:
        raise ZeroDivisionError("singular row system")
    return Y


def crank_nicolson(ms, as_, dt, F, nsteps=None):
    """C restatement of crank_nicolson (stk/cn_baseline.hpp:26-48), banded Cholesky."""
    ndim = len(ms)
    F = np.ascontiguousarray(F, dtype=np.float64)
    nsteps = F.shape[0] if nsteps is None else nsteps
    n = (C.c_int64 * 3)(*[m[0].size for m in ms], *([1] * (3 - ndim)))
    keep = []
    U = np.empty((nsteps, F.shape[1]))
    st = clib.or_crank_nicolson(ndim, n, nsteps, dt, _arr_pp([m[0] for m in ms], keep),
                                _arr_pp([m[1] for m in ms], keep),
                                _arr_pp([a[0] for a in as_], keep),
                                _arr_pp([a[1] for a in as_], keep), _p(F), _p(U))
    if st:
        raise np.linalg.LinAlgError("crank_nicolson: not s.p.d.")
    return U


# -------------------------------------------------------------------- heat (numpy) --
def p1_pencil_eig(m, a):
    """Numerical sym_gen_eig(A, M) of a 1D pencil by scipy (independent of the closed form)."""
    import scipy.linalg as sl
    lam, X = sl.eigh(tri_dense(a), tri_dense(m))
    return lam, X


def heat_decoupled(eigs, d, c, F, nsteps=None):
    """solve_projected_heat_with (stk/sylvester.hpp:117-142) in tensor form with numpy:
    per-axis transforms G~ = (X_x (x) X_y (x) X_z)^T F, per-mode recurrence, inverse.
    ``eigs`` = [(lam, X)] per axis; F is (nt, nx) C-order; nsteps => causal prefix."""
    ns = [e[0].size for e in eigs]
    nt = F.shape[0] if nsteps is None else nsteps
    G = np.asarray(F[:nt], dtype=np.float64).reshape(nt, *ns)
    for ax, (lam, X) in enumerate(eigs):  # forward: contract axis ax+1 with X
        G = np.moveaxis(np.tensordot(G, X, axes=([ax + 1], [0])), -1, ax + 1)
    lam_t = np.zeros(ns)
    for ax, (lam, X) in enumerate(eigs):
        shape = [1] * len(ns)
        shape[ax] = ns[ax]
        lam_t = lam_t + lam.reshape(shape)
    Y = np.empty_like(G)
    y = np.zeros(ns)
    for j in range(nt):
        piv = d[0][j] + lam_t * c[0][j]
        rhs = G[j]
        if j > 0:
            rhs = rhs - (d[1][j - 1] + lam_t * c[1][j - 1]) * y
        y = rhs / piv
        Y[j] = y
    for ax, (lam, X) in enumerate(eigs):
        Y = np.moveaxis(np.tensordot(Y, X, axes=([ax + 1], [1])), -1, ax + 1)
    return Y.reshape(nt, -1)


def toeplitz_tridiag_solve_images(a, b, r):
    """Solve tridiag(a, b, a) x = r along axis 0 of r (shape (n, cols); a, b of shape (cols,),
    b > 2|a|) by the method of images: the restriction of the bi-infinite Toeplitz operator
    (constant pivot w = (b + sqrt(b^2 - 4a^2))/2, q = -a/w) to odd 2N-periodic sequences is a
    causal and an anti-causal first-order recurrence with the constant coefficient q whose
    start values follow from two weighted totals -- the arithmetic of
    csrc/heat_tridiag.cuh::heat_tridiag_tma_kernel, unchunked."""
    n = r.shape[0]
    N = n + 1
    sq = np.sqrt((b + 2.0 * a) * (b - 2.0 * a))
    q = -a / (0.5 * (b + sq))
    gam = 1.0 / sq
    A = np.empty_like(r)
    acc = np.zeros_like(a)
    for i in range(n):
        acc = r[i] + q * acc
        A[i] = acc
    aN = q * acc                       # zero-start causal total at the mirror row N
    acc = np.zeros_like(a)
    for i in range(n - 1, -1, -1):
        acc = r[i] + q * acc
    b0 = q * acc                       # zero-start anti-causal total at the mirror row 0
    qN = q ** N
    A0 = (qN * aN - b0) / (1.0 - qN * qN)
    BN = -(qN * A0 + aN)
    A += (q[None, :] ** np.arange(1, n + 1)[:, None]) * A0
    x = np.empty_like(r)
    Bn = BN
    for i in range(n - 1, -1, -1):
        x[i] = gam * (A[i] + q * Bn)
        Bn = r[i] + q * Bn
    return x


def heat_line_march(eigs_fast, m0, a0, d, c, F, nsteps=None):
    """solve_projected_heat_with (stk/sylvester.hpp:117-142) with axis 0 left untransformed:
    the faster axes are diagonalised by ``eigs_fast`` = [(lam, X)] (X^T M X = I), and each step
    of the temporal recurrence is, per column, one symmetric Toeplitz tridiagonal solve along
    axis 0,  [(d_l + lam_c c_l) M_0 + c_l A_0] z_l = g_l - [(d^s + lam_c c^s) M_0 + c^s A_0]
    z_{l-1}  (m0, a0 = the 1D P1 factors of axis 0, uniform grid).  Equal to heat_decoupled in
    exact arithmetic; restates the line-solve schedule of csrc/heat_tridiag.cuh."""
    n0 = m0[0].size
    ns = [e[0].size for e in eigs_fast]
    nt = F.shape[0] if nsteps is None else nsteps
    G = np.asarray(F[:nt], dtype=np.float64).reshape(nt, n0, *ns)
    for ax, (lam, X) in enumerate(eigs_fast):
        G = np.moveaxis(np.tensordot(G, X, axes=([ax + 2], [0])), -1, ax + 2)
    lam_c = np.zeros(ns)
    for ax, (lam, X) in enumerate(eigs_fast):
        shape = [1] * len(ns)
        shape[ax] = ns[ax]
        lam_c = lam_c + lam.reshape(shape)
    lam_c = lam_c.reshape(-1)
    G = G.reshape(nt, n0, -1)
    md, mo, ad, ao = m0[0][0], m0[1][0], a0[0][0], a0[1][0]
    assert np.allclose(m0[0], md) and np.allclose(m0[1], mo) and np.allclose(a0[0], ad) \
        and np.allclose(a0[1], ao), "axis 0 must be a uniform P1 axis (Toeplitz factors)"
    Z = np.empty_like(G)
    z = np.zeros_like(G[0])
    for l in range(nt):
        p = d[0][l] + lam_c * c[0][l]
        rhs = G[l]
        if l > 0:
            pp = d[1][l - 1] + lam_c * c[1][l - 1]
            sa, sb = pp * mo + c[1][l - 1] * ao, pp * md + c[1][l - 1] * ad
            zz = np.zeros((n0 + 2, z.shape[1]))
            zz[1:-1] = z
            rhs = rhs - (sb * z + sa * (zz[:-2] + zz[2:]))
        z = toeplitz_tridiag_solve_images(p * mo + c[0][l] * ao, p * md + c[0][l] * ad, rhs)
        Z[l] = z
    Z = Z.reshape(nt, n0, *ns)
    for ax, (lam, X) in enumerate(eigs_fast):
        Z = np.moveaxis(np.tensordot(Z, X, axes=([ax + 2], [1])), -1, ax + 2)
    return Z.reshape(nt, -1)


class DecoupledStream:
    """heat_decoupled over consecutive time chunks: the same tensor-form
    solve_projected_heat_with (stk/sylvester.hpp:117-142), with the per-mode recurrence
    state y_{j0-1} carried from one chunk to the next, so a full n_t solve can be run (and
    compared, or timed) a bounded number of time slices at a time.  step(F_chunk) takes the
    next (k, n_x) C-order rows of F and returns the same rows of U."""

    def __init__(self, eigs, d, c):
        self.eigs = eigs
        self.d, self.c = d, c
        self.ns = [e[0].size for e in eigs]
        lam_t = np.zeros(self.ns)
        for ax, (lam, X) in enumerate(eigs):
            shape = [1] * len(self.ns)
            shape[ax] = self.ns[ax]
            lam_t = lam_t + lam.reshape(shape)
        self.lam_t = lam_t
        self.j = 0
        self.y = np.zeros(self.ns)

    def step(self, F):
        k = F.shape[0]
        G = np.asarray(F, dtype=np.float64).reshape(k, *self.ns)
        for ax, (lam, X) in enumerate(self.eigs):
            G = np.moveaxis(np.tensordot(G, X, axes=([ax + 1], [0])), -1, ax + 1)
        d, c, lam_t, y = self.d, self.c, self.lam_t, self.y
        for i in range(k):
            j = self.j + i
            rhs = G[i]
            if j > 0:
                rhs = rhs - (d[1][j - 1] + lam_t * c[1][j - 1]) * y
            y = rhs / (d[0][j] + lam_t * c[0][j])
            G[i] = y
        self.y, self.j = y, self.j + k
        for ax, (lam, X) in enumerate(self.eigs):
            G = np.moveaxis(np.tensordot(G, X, axes=([ax + 1], [1])), -1, ax + 1)
        return G.reshape(k, -1)


def crank_nicolson_splu(ms, as_, dt, F, nsteps=None):
    """CN (stk/cn_baseline.hpp:26-48) with scipy SuperLU in place of SimplicialLLT."""
    import scipy.sparse.linalg as spl
    M, A = tensor_sparse(ms, as_)
    lhs = (M + (dt / 2.0) * A).tocsc()
    rhs = (M - (dt / 2.0) * A).tocsr()
    lu = spl.splu(lhs)
    nt = F.shape[0] if nsteps is None else nsteps
    U = np.empty((nt, F.shape[1]))
    u = np.zeros(F.shape[1])
    for l in range(nt):
        u = lu.solve(rhs @ u + F[l])
        U[l] = u
    return U


def heat_residual(ms, as_, d, c, U, F):
    """||F - KronOp::apply(U)||_F / ||F||_F (stk/bench.hpp:508)."""
    R = F - heat_apply(ms, as_, d, c, U)
    return float(np.linalg.norm(R) / np.linalg.norm(F))


# ------------------------------------------------------------------------------ wave --
def ref_lib():
    so = HERE / "_ref" / "libstkref.so"
    if not so.exists():
        if (Path("/root/reference/proj/include/stk/splines.hpp")).exists():
            subprocess.run(["make", "-C", str(HERE), "ref"], check=True, capture_output=True)
        else:
            return None
    lib = C.CDLL(str(so))
    lib.ref_wave_space_bands.argtypes = [C.c_double, C.c_double, C.c_int, C.c_int, _dp]
    lib.ref_wave_time_bands.argtypes = [C.c_int, C.c_double, C.c_int, _dp]
    lib.ref_gauss_legendre.argtypes = [C.c_int, C.c_double, C.c_double, _dp, _dp]
    lib.ref_spline_eval.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                    C.c_double, C.c_int, _dp]
    return lib


def ref_wave_bands(nh: int, nt: int, degree: int = 3, T: float = 1.0):
    """(space [M|A|Q], time [Q|D|M]) bands from the reference's own spline code."""
    lib = ref_lib()
    if lib is None:
        raise FileNotFoundError("oracle/_ref not built and reference tree absent")
    sb = np.zeros(3 * 7 * nh)
    ntb = nt + degree - 2
    tb = np.zeros(3 * 7 * ntb)
    assert lib.ref_wave_space_bands(0.0, 1.0, nh, degree, _p(sb)) == nh
    assert lib.ref_wave_time_bands(nt, T, degree, _p(tb)) == ntb
    return sb.reshape(3, 7, nh), tb.reshape(3, 7, ntb)


def band_dense(band):
    n = band.shape[1]
    m = np.zeros((n, n))
    for dd in range(7):
        for i in range(n):
            j = i + dd - 3
            if 0 <= j < n:
                m[i, j] = band[dd, i]
    return m


def band_sparse(band):
    import scipy.sparse as sp
    n = band.shape[1]
    rows, cols, vals = [], [], []
    for dd in range(7):
        i = np.arange(n)
        j = i + dd - 3
        ok = (j >= 0) & (j < n)
        rows.append(i[ok]); cols.append(j[ok]); vals.append(band[dd][ok])
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(n, n))


def wave_apply(sb, tb, U):
    """C restatement of WaveOperator::apply; U is (nt, nh) C-order (== nh x nt col-major)."""
    nt, nh = U.shape
    U = np.ascontiguousarray(U, dtype=np.float64)
    out = np.empty_like(U)
    clib.or_wave_apply(nh, nt, _p(np.ascontiguousarray(sb).ravel()),
                       _p(np.ascontiguousarray(tb).ravel()), _p(U), _p(out))
    return out


def band_transpose(band):
    """Band of A^T from the 7-band storage of A (band[d, i] = A(i, i + d - 3))."""
    n = band.shape[1]
    out = np.zeros_like(band)
    for d in range(7):
        o = d - 3
        i0, i1 = max(0, -o), min(n, n - o)
        out[d, i0:i1] = band[3 - o, i0 + o:i1 + o]
    return out


def band_rows(band, U):
    """A U for a 7-band A, every product and sum in U's dtype (rows of U = columns of A)."""
    n = band.shape[1]
    out = np.zeros_like(U)
    for d in range(7):
        o = d - 3
        i0, i1 = max(0, -o), min(n, n - o)
        out[i0:i1] += band[d, i0:i1, None].astype(U.dtype) * U[i0 + o:i1 + o]
    return out


def wave_residual_banded(sb, tb, b, xh, xl=None, dtype=np.longdouble):
    """b - B (x_h + x_l) with WaveOperator::apply (stk/outer_krylov.hpp:178-186:
    vec(M_h U Q_t^T + A_h U (D_t + D_t^T) + Q_h U M_t), U = x as n_h x n_t column-major)
    evaluated band by band in `dtype` (numpy longdouble: 64-bit mantissa), O(49 N) -- the
    extended-precision check of the GPU's double-double residual at full config-4 size.
    Returns the residual vector (dtype)."""
    nh, nt = sb.shape[2], tb.shape[2]
    x = xh.astype(dtype) + (0 if xl is None else xl.astype(dtype))
    U = x.reshape(nt, nh).T
    Mh, Ah, Qh = sb
    Qt, Dt, Mt = tb
    E = Dt + band_transpose(Dt)  # formed in FP64, as the reference's sparse sum is
    out = band_rows(Qt, band_rows(Mh, U).T).T
    out += band_rows(E, band_rows(Ah, U).T).T  # U E = (E^T U^T)^T, E = E^T
    out += band_rows(band_transpose(Mt), band_rows(Qh, U).T).T
    return b.astype(dtype) - out.T.ravel()


def wave_residual_floor(sb, tb, b, xh, xl=None, unit=2.0 ** -63):
    """Rounding floor of wave_residual_banded: unit x || |S_p| |U| |T_p|^T || / ||b|| -- the
    size of the terms the extended-precision evaluation cancels, times its unit roundoff."""
    ab = lambda a: np.abs(a)  # noqa: E731
    x = np.abs(xh) + (0 if xl is None else np.abs(xl))
    r = wave_residual_banded(ab(sb), ab(tb), np.zeros_like(b), x, dtype=np.float64)
    return unit * float(np.linalg.norm(r)) / float(np.linalg.norm(b))


def wave_residual_exact_entries(sb, tb, b, xh, xl, idx):
    """b_i - (B x)_i for the listed vec indices i, exactly (Python Fractions: every band
    product and sum exact, x = x_hi + x_lo exact), with E = D_t + D_t^T rounded in FP64 as the
    reference forms it.  Returns (r_i rounded to double, sum of |terms|) per index."""
    from fractions import Fraction as Fr
    nh, nt = sb.shape[2], tb.shape[2]
    Mh, Ah, Qh = sb
    Qt, Dt, Mt = tb
    E = Dt + band_transpose(Dt)

    def S(k, i, a):  # S_k(i, a)
        o = a - i
        return float(sb[k][o + 3][i]) if -3 <= o <= 3 and 0 <= a < nh else 0.0

    def band(m, i, j):  # m(i, j) for a time band
        o = j - i
        return float(m[o + 3][i]) if -3 <= o <= 3 and 0 <= j < nt else 0.0

    out = []
    for g in idx:
        ih, it = g % nh, g // nh
        acc = Fr(float(b[g]))
        mag = abs(float(b[g]))
        for a in range(max(0, ih - 3), min(nh, ih + 4)):
            for bb in range(max(0, it - 3), min(nt, it + 4)):
                u = Fr(float(xh[a + nh * bb])) + Fr(float(xl[a + nh * bb]))
                # M_h U Q_t^T: Mh(ih,a) Qt(it,bb); A_h U E: Ah(ih,a) E(bb,it); Q_h U M_t: Qh(ih,a) Mt(bb,it)
                for sv, tv in ((S(0, ih, a), band(Qt, it, bb)), (S(1, ih, a), band(E, bb, it)),
                               (S(2, ih, a), band(Mt, bb, it))):
                    if sv != 0.0 and tv != 0.0:
                        term = Fr(sv) * Fr(tv) * u
                        acc -= term
                        mag += abs(float(term))
        out.append((float(acc), mag))
    return out


def wave_refined_direct(sb, tb, b, steps=3):
    """kron_direct_solve (stk/bench.hpp:414-429, SuperLU) followed by `steps` rounds of
    iterative refinement with the longdouble banded residual: the oracle solution for
    forward-error checks of the GPU's refined solve.  Returns (x_hi, x_lo, relres history)."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    Mh, Ah, Qh = (band_sparse(sb[k]) for k in range(3))
    Qt, Dt, Mt = (band_sparse(tb[k]) for k in range(3))
    E = (Dt + Dt.T).tocsr()
    lu = spl.splu((sp.kron(Qt, Mh) + sp.kron(E.T, Ah) + sp.kron(Mt.T, Qh)).tocsc())
    L = np.longdouble
    xh = lu.solve(b)
    xl = np.zeros_like(xh)
    bn = float(np.linalg.norm(b))
    hist = []
    for _ in range(steps):
        r = wave_residual_banded(sb, tb, b, xh, xl)
        hist.append(float(np.sqrt(np.sum(r * r))) / bn)
        s = xh.astype(L) + xl.astype(L) + lu.solve(r.astype(np.float64)).astype(L)
        xh = s.astype(np.float64)
        xl = (s - xh.astype(L)).astype(np.float64)
    r = wave_residual_banded(sb, tb, b, xh, xl)
    hist.append(float(np.sqrt(np.sum(r * r))) / bn)
    return xh, xl, hist


class WaveSystemNP:
    """numpy/scipy restatement of the wave system: WaveOperator (stk/outer_krylov.hpp:
    168-191), TwoTermPrecond (stk/sylvester.hpp:153-181, scipy eigh) and gmres (:75-164)."""

    def __init__(self, sb, tb):
        import scipy.linalg as sl
        self.Mh, self.Ah, self.Qh = (band_sparse(sb[k]) for k in range(3))
        self.Qt, self.Dt, self.Mt = (band_sparse(tb[k]) for k in range(3))
        self.E = (self.Dt + self.Dt.T).tocsr()
        self.nh, self.nt = sb.shape[2], tb.shape[2]
        self.lam, self.Xs = sl.eigh(self.Qh.toarray(), self.Mh.toarray())
        self.theta, self.Xt = sl.eigh(self.Qt.toarray(), self.Mt.toarray())

    def apply(self, x):
        U = x.reshape(self.nt, self.nh).T  # nh x nt view (column-major vec)
        out = (self.Mh @ U) @ self.Qt.T + (self.Ah @ U) @ self.E + (self.Qh @ U) @ self.Mt
        return np.ascontiguousarray(out.T).ravel()

    def precond(self, v):
        V = v.reshape(self.nt, self.nh).T
        wt = self.Xs.T @ V @ self.Xt
        wt = wt / (self.lam[:, None] + self.theta[None, :])
        W = self.Xs @ wt @ self.Xt.T
        return np.ascontiguousarray(W.T).ravel()

    def gmres(self, b, tol=1e-8, maxit=200):
        """Right-preconditioned full GMRES, MGS + one re-orth pass, Givens (reference)."""
        norm_b = np.linalg.norm(b)
        x = np.zeros_like(b)
        if norm_b == 0:
            return x, 0, []
        r = b.copy()
        beta = np.linalg.norm(r)
        basis = [r / beta]
        hcols = []
        g = np.zeros(maxit + 1)
        g[0] = beta
        cs, sn = [], []
        hist = []
        k = 0
        total = 0
        for j in range(maxit):
            w = self.apply(self.precond(basis[j]))
            col = np.zeros(j + 2)
            for i in range(j + 1):
                hij = basis[i] @ w
                w -= hij * basis[i]
                col[i] = hij
            for i in range(j + 1):
                corr = basis[i] @ w
                w -= corr * basis[i]
                col[i] += corr
            hlast = np.linalg.norm(w)
            col[j + 1] = hlast
            for i in range(j):
                t = cs[i] * col[i] + sn[i] * col[i + 1]
                col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1]
                col[i] = t
            a, bb = col[j], col[j + 1]
            rr = np.hypot(a, bb)
            cc = 1.0 if rr == 0 else a / rr
            ss = 0.0 if rr == 0 else bb / rr
            cs.append(cc); sn.append(ss)
            col[j], col[j + 1] = rr, 0.0
            t = cc * g[j] + ss * g[j + 1]
            g[j + 1] = -ss * g[j] + cc * g[j + 1]
            g[j] = t
            hcols.append(col)
            relres = abs(g[j + 1]) / norm_b
            hist.append(relres)
            k = j + 1
            total = j + 1
            if relres <= tol or hlast == 0:
                break
            basis.append(w / hlast)
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            acc = g[i]
            for jj in range(i + 1, k):
                acc -= hcols[jj][i] * y[jj]
            y[i] = acc / hcols[i][i]
        xk = sum(y[i] * basis[i] for i in range(k))
        x += self.precond(xk)
        return x, total, hist

    def modal_banded(self, v):
        """The space-modal time-banded preconditioner (product: stkg_modal_banded_solve,
        DESIGN.md K2d) restated densely: a_i = (X_s^T A_h X_s)_ii, K_i = sym(Q_t + a_i E +
        lambda_i M_t), W = X_s [rows i of X_s^T V solved with K_i]."""
        import scipy.linalg as sl
        V = v.reshape(self.nt, self.nh).T
        a = np.einsum("ri,rc,ci->i", self.Xs, self.Ah.toarray(), self.Xs)
        Qt, Mt, E = self.Qt.toarray(), self.Mt.toarray(), self.E.toarray()
        Vt = self.Xs.T @ V
        Wt = np.empty_like(Vt)
        for i in range(self.nh):
            K = Qt + a[i] * E + self.lam[i] * Mt
            Wt[i] = sl.solve(0.5 * (K + K.T), Vt[i], assume_a="pos")
        return (self.Xs @ Wt).T.ravel()

    def modal_banded_apply(self, w):
        """P w for the modal banded preconditioner's operator (the wave operator with A_h
        replaced by A' = M_h X_s diag(a) X_s^T M_h): the backward-error check of P^-1."""
        U = w.reshape(self.nt, self.nh).T
        a = np.einsum("ri,rc,ci->i", self.Xs, self.Ah.toarray(), self.Xs)
        MX = self.Mh @ self.Xs
        Ap = (MX * a[None, :]) @ MX.T
        out = (self.Mh @ U) @ self.Qt.T + (Ap @ U) @ self.E + (self.Qh @ U) @ self.Mt
        return out.T.ravel()

    def direct(self, b):
        """kron_direct_solve (stk/bench.hpp:414-429) with scipy SuperLU: sum_p D_p (x) A_p."""
        import scipy.sparse as sp
        import scipy.sparse.linalg as spl
        B = (sp.kron(self.Qt, self.Mh) + sp.kron(self.E.T, self.Ah) + sp.kron(self.Mt.T, self.Qh))
        return spl.splu(B.tocsc()).solve(b)


# ----------------------------------------------------------------- load projection --
def gauss_legendre01(npoints: int):
    """gauss_legendre(npoints, 0, 1) (stk/quadrature.hpp:17-64): the reference's own rule
    (compiled from the reference by oracle/_ref, committed as tests/golden/wave_bands_ref.npz
    by tests/golden/make_golden.py) when the fixture holds it, else numpy's Golub-Welsch rule
    (agrees to a few ulps; tests/test_host_cpu.py pins both)."""
    fx = HERE.parent / "tests" / "golden" / "wave_bands_ref.npz"
    if fx.exists():
        z = np.load(fx)
        if f"gauss_{npoints}_x" in z:
            return z[f"gauss_{npoints}_x"], z[f"gauss_{npoints}_w"]
    x, w = np.polynomial.legendre.leggauss(npoints)
    return (x + 1.0) / 2.0, w / 2.0


def project_rhs_heat(theta, f, nt: int, T: float, a: float, b: float, nh: int,
                     trapezoidal_time: bool = False, npoints: int = 6, rule=None):
    """project_rhs_heat (stk/rhs_sep.hpp:111-151) for one separable term theta(t) f(x),
    with the reference's summation order: H[l] = sum_i dt w_i theta(t_l + dt x_i) (or the
    trapezoid dt/2 (theta(t_l) + theta(t_l+1))), and G[j] accumulates the rising-hat part of
    element j and then the falling-hat part of element j+1.  Returns (G (nh,), H (nt,))."""
    xs, ws = rule if rule is not None else gauss_legendre01(npoints)
    dt = T / nt  # TimeGrid::dt (stk/discretize.hpp:13-24), node(l) = l * dt
    t0 = np.arange(nt) * dt
    t1 = np.arange(1, nt + 1) * dt
    H = np.zeros(nt)
    if trapezoidal_time:
        H = dt / 2.0 * (theta(t0) + theta(t1))
    else:
        for xi, wi in zip(xs, ws):
            H = H + dt * wi * theta(t0 + dt * xi)
    h = (b - a) / (nh + 1)  # SpaceGrid1D::fem_h
    x0 = a + np.arange(nh + 1) * h  # element e = [x0[e], x0[e] + h]
    G = np.zeros(nh)
    for xi, wi in zip(xs, ws):  # rising part of element e -> node e+1 -> G[e], e < nh
        x = x0[:nh] + h * xi
        G = G + (h * wi) * f(x) * ((x - x0[:nh]) / h)
    for xi, wi in zip(xs, ws):  # falling part of element e -> node e -> G[e-1], e >= 1
        x = x0[1:] + h * xi
        G = G + (h * wi) * f(x) * (1.0 - (x - x0[1:]) / h)
    return G, H


def heat_ex1_theta(t):
    """heat_ex1_rhs theta (stk/bench.hpp:300-306): 10 sin(t) t."""
    return 10.0 * np.sin(t) * t


def heat_ex1_f(x):
    """heat_ex1_rhs f_x = f_y: cos(pi x / 2) (stk/bench.hpp:300-306)."""
    return np.cos(np.pi / 2.0 * x)


def heat_ex1_load(ndim: int, nh: int, nt: int, T: float = 10.0,
                  trapezoidal_time: bool = False):
    """assemble_heat's built-in heat-ex1 load (stk/bench.hpp:361-406) on Omega = (-1,1)^ndim:
    F = L H^T with L = kron_cols(G_x, G_y) (index ix*ny + iy, :378-384), H the temporal
    factor of the x-term (trapezoidal when requested; the y-term is projected with the
    quadrature mode and contributes only its spatial factor, :375-385).  3D (no reference
    function) extends the same product.  Returns (L (n_x,), H (nt,))."""
    G, H = project_rhs_heat(heat_ex1_theta, heat_ex1_f, nt, T, -1.0, 1.0, nh, trapezoidal_time)
    L = G
    for _ in range(ndim - 1):
        L = np.kron(L, G)
    return L, H


# ----------------------------------------------------------------------- generator --
def fill_uniform(count, seed, stream, offset=0):
    out = np.empty(count)
    clib.or_fill_uniform(_p(out), count, seed, stream, offset)
    return out


# ------------------------------------------------------------------------------ RKSM --
def adaptive_next_shift(shifts, ritz, lam_min, lam_max):
    """adaptive_next_shift (stk/rksm.hpp:67-102)."""
    n = 200
    lo, hi = np.log(lam_min / 2.0), np.log(2.0 * lam_max)
    best, best_val = None, -np.inf
    for i in range(n):
        x = -np.exp(lo + (hi - lo) * i / (n - 1))
        if best is None:
            best = x
        val = 0.0
        for s in shifts:
            d = abs(x - s)
            if d == 0.0:
                val = -np.inf
                break
            val += np.log(d)
        for lam in ritz:
            val -= np.log(max(abs(x + lam), 1e-300))
        if val > best_val or (val == best_val and abs(x) < abs(best)):
            best_val, best = val, x
    return best


def _colpiv_qr(A, threshold):
    """Rank-revealing column-pivoted Householder QR (Eigen ColPivHouseholderQR semantics):
    returns Q (n x rank), R (rank x m) in the original column order."""
    import scipy.linalg as sl
    Q, R, piv = sl.qr(A, mode="economic", pivoting=True)
    d = np.abs(np.diag(R))
    rank = int(np.sum(d > threshold * d[0])) if d.size and d[0] > 0 else 0
    Rorig = np.zeros((rank, A.shape[1]))
    Rorig[:, piv] = R[:rank]
    return Q[:, :rank], Rorig


def lowrank_norm(left, right):
    """lowrank_norm (stk/la_core.hpp:114-119): thin QR of both factors."""
    if left.shape[1] == 0:
        return 0.0
    r1 = np.linalg.qr(left, mode="r")
    r2 = np.linalg.qr(right, mode="r")
    return float(np.linalg.norm(r1 @ r2.T))


def rksm_solve(ms, as_, d, c, L, R, tol=1e-8, maxit=100, trunc_tol=1e-10, fixed_iters=0):
    """rksm_solve (stk/rksm.hpp:127-234) restated with scipy: SuperLU in place of the
    cached SimplicialLLT shifted factors, pivoted Householder QR (scipy) in place of
    ColPivHouseholderQR, scipy eigh for sym_gen_eig.  The spectral interval is the exact
    one of the tensor pencil widened by [1/2, 2] (the product does the same; the
    reference estimates it by 30 power/inverse iterations, :21-51).
    L: n x r, R: nt x r.  Returns (left, right, iterations, history)."""
    import scipy.linalg as sl
    import scipy.sparse.linalg as spl
    M, A = tensor_sparse(ms, as_)
    M, A = M.tocsc(), A.tocsc()
    n, nt = M.shape[0], R.shape[0]
    Dm, Cm = bidiag_dense(d), bidiag_dense(c)
    norm_f = lowrank_norm(L, R)
    if norm_f == 0:
        return np.zeros((n, 0)), np.zeros((nt, 0)), 0, []
    f1, r_thin = _colpiv_qr(L, 1e-13)
    rf = f1.shape[1]
    f2 = R @ r_thin.T
    lam1 = [sl.eigh(tri_dense(a), tri_dense(m), eigvals_only=True) for m, a in zip(ms, as_)]
    lam_min = sum(x.min() for x in lam1) / 2.0
    lam_max = 2.0 * sum(x.max() for x in lam1)
    V = f1.copy()
    newest = f1.copy()
    shifts, ritz, hist = [], [], []
    y = None
    it = 0
    total = fixed_iters if fixed_iters > 0 else maxit
    for it in range(1, total + 1):
        k = V.shape[1]
        hm = V.T @ (M @ V)
        ha = V.T @ (A @ V)
        hm = 0.5 * (hm + hm.T)
        ha = 0.5 * (ha + ha.T)
        lam, X = sl.eigh(ha, hm)
        ritz = lam
        g = (V.T @ f1) @ f2.T
        y = solve_projected_heat_with_dense(X, lam, d, c, np.ascontiguousarray(g.T)).T  # k x nt
        left = np.hstack([L, M @ V, A @ V])
        right = np.hstack([R, -(Dm.T @ y.T), -(Cm.T @ y.T)])
        relres = lowrank_norm(left, right) / norm_f
        hist.append(relres)
        if (fixed_iters <= 0 and relres <= tol) or it == total:
            break
        sigma = -lam_max if not shifts else adaptive_next_shift(shifts, ritz, lam_min, lam_max)
        shifts.append(sigma)
        w = spl.splu((A - sigma * M).tocsc()).solve(M @ newest)
        for _ in range(2):
            w = w - V @ (V.T @ w)
        wq, _ = _colpiv_qr(w, 1e-12)
        if wq.shape[1] == 0:
            break
        V = np.hstack([V, wq])
        newest = wq
    tol = trunc_tol if fixed_iters > 0 else tol
    # lowrank_truncate(V, y^T, tol) (stk/la_core.hpp:134-162)
    q1, r1 = np.linalg.qr(V)
    q2, r2 = np.linalg.qr(y.T)
    U_, s, Vt = np.linalg.svd(r1 @ r2.T)
    total2 = np.sum(s ** 2)
    keep = s.size
    tail2 = 0.0
    while keep > 0:
        nxt = tail2 + s[keep - 1] ** 2
        if nxt > tol * tol * total2:
            break
        tail2 = nxt
        keep -= 1
    left = q1 @ U_[:, :keep] * s[:keep]
    right = q2 @ Vt[:keep].T
    return left, right, it, hist
