"""Error behaviour of the C ABI and its bindings, mirroring the reference's error classes
(stk/errors.hpp:9-42) and the precondition checks of the functions each entry point
replaces.  The argument checks run before any CUDA call, so most cases need no GPU; the
ones that need a live plan are marked gpu."""
import ctypes as C

import numpy as np
import pytest


def _desc_1d(stk, n=15, nt=4, transform=0, p1h=0.0625):
    from paper_1912_10082_b200._lib import HeatDesc
    keep = []

    def arr(a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        keep.append(a)
        return a.ctypes.data_as(C.POINTER(C.c_double))

    e = stk.p1_eigpair(stk.SpaceGrid1D(0.0, 1.0, n))
    D, Cm = stk.heat_time_matrices(stk.TimeGrid(nt, 1.0))
    d = HeatDesc()
    d.ndim = 1
    d.n[0], d.n[1], d.n[2] = n, 1, 1
    d.nt = nt
    d.d_diag, d.c_diag = arr(D.diag), arr(Cm.diag)
    d.d_sup = arr(D.sup if D.sup.size else np.zeros(1))
    d.c_sup = arr(Cm.sup if Cm.sup.size else np.zeros(1))
    d.X[0] = arr(np.asfortranarray(e.X))
    d.lambdas[0] = arr(e.lambdas)
    d.transform = transform
    d.p1_h[0] = p1h
    return d, keep


def _create(desc):
    from paper_1912_10082_b200._lib import lib
    h = C.c_void_p()
    st = lib.stkg_heat_create(C.byref(h), C.byref(desc), None)
    return st, h


def _msg():
    from paper_1912_10082_b200._lib import lib
    return lib.stkg_last_error_message().decode()


def test_heat_create_argument_errors(stk):
    from paper_1912_10082_b200.errors import STKG_ARGUMENT
    d, keep = _desc_1d(stk)
    d.ndim = 4
    st, _ = _create(d)
    assert st == STKG_ARGUMENT and "ndim must be 1, 2 or 3" in _msg()
    d, keep = _desc_1d(stk)
    d.nt = 0
    st, _ = _create(d)
    assert st == STKG_ARGUMENT and "nt must be >= 1" in _msg()
    d, keep = _desc_1d(stk, n=14, transform=1)  # n + 1 = 15: not a power of two
    st, _ = _create(d)
    assert st == STKG_ARGUMENT and "power of two" in _msg()
    d, keep = _desc_1d(stk, transform=1, p1h=0.0)
    st, _ = _create(d)
    assert st == STKG_ARGUMENT and "p1_h" in _msg()
    d, keep = _desc_1d(stk)
    d.transform = 7
    st, _ = _create(d)
    assert st == STKG_ARGUMENT and "unknown transform" in _msg()
    d, keep = _desc_1d(stk)
    d.lambdas[0] = None
    st, _ = _create(d)
    assert st == STKG_ARGUMENT and "missing EigPair" in _msg()


def test_null_handles_are_argument_errors(stk):
    from paper_1912_10082_b200._lib import lib, RksmOpts
    from paper_1912_10082_b200.errors import STKG_ARGUMENT
    null = C.c_void_p()
    assert lib.stkg_heat_solve(null, null, null) == STKG_ARGUMENT
    assert lib.stkg_heat_apply(null, null, null) == STKG_ARGUMENT
    assert lib.stkg_wave_apply(null, null, null) == STKG_ARGUMENT
    assert lib.stkg_two_term_solve(null, null, null) == STKG_ARGUMENT
    rk = C.c_int64()
    assert lib.stkg_heat_rksm(null, 1, null, null, C.byref(RksmOpts(1e-8, 10, 0, 1e-10)),
                              null, null, 4, C.byref(rk), None) == STKG_ARGUMENT
    assert "null argument" in _msg()


def test_python_layer_argument_errors(stk):
    e = stk.p1_eigpair(stk.SpaceGrid1D(0.0, 1.0, 7))
    D, Cm = stk.heat_time_matrices(stk.TimeGrid(4, 1.0))
    D5, _ = stk.heat_time_matrices(stk.TimeGrid(5, 1.0))
    with pytest.raises(stk.ArgumentError, match="1 to 3 spatial axes"):
        stk.HeatPlan(stk.TensorEigPair([e] * 4), D, Cm)
    with pytest.raises(stk.ArgumentError, match="D and C sizes differ"):
        stk.HeatPlan(e, D5, Cm)
    with pytest.raises(stk.ArgumentError, match="transform"):
        stk.HeatPlan(e, D, Cm, transform="fft")
    with pytest.raises(stk.ArgumentError, match="p1_h"):
        stk.HeatPlan(e, D, Cm, transform="dst")


def test_wave_create_argument_errors(stk):
    from paper_1912_10082_b200._lib import WaveDesc, lib
    from paper_1912_10082_b200.errors import STKG_ARGUMENT
    d = WaveDesc()
    d.nh, d.nt = 0, 4
    h = C.c_void_p()
    assert lib.stkg_wave_create(C.byref(h), C.byref(d), None) == STKG_ARGUMENT
    assert "bad sizes" in _msg()
    d.nh = 4
    assert lib.stkg_wave_create(C.byref(h), C.byref(d), None) == STKG_ARGUMENT
    assert "missing bands" in _msg()


def test_error_message_is_thread_local(stk):
    """stkg_last_error_message is per thread (errors.cpp): a failing call on one thread does
    not overwrite another thread's message."""
    import threading
    from paper_1912_10082_b200._lib import lib
    z = np.zeros(4)
    p = z.ctypes.data_as(C.POINTER(C.c_double))
    lib.stkg_heat_time_matrices(0, 1.0, p, p, p, p)
    mine = _msg()
    seen = []

    def other():
        lib.stkg_fem1d_matrices(0.0, 1.0, 0, p, p, p, p)
        seen.append(_msg())

    t = threading.Thread(target=other)
    t.start()
    t.join()
    assert "nt must be >= 1" in mine and _msg() == mine
    assert seen and seen[0] != mine


# ---------------------------------------------------------------------- with a GPU --
@pytest.mark.gpu
def test_plan_level_errors(stk, cuda):
    import torch
    plan = stk.HeatPlan.p1_uniform(1, 15, 4, with_operator=False)
    F = torch.zeros((4, 15), dtype=torch.float64, device="cuda")
    with pytest.raises(stk.ArgumentError, match="without the spatial factors"):
        plan.apply(F)
    with pytest.raises(stk.ArgumentError, match="alias"):
        plan.solve(F, out=F)
    big = torch.zeros((5, 15), dtype=torch.float64, device="cuda")  # partial overlap
    with pytest.raises(stk.ArgumentError, match="alias"):
        plan.solve(big[:4], out=big[1:])
    p2 = stk.HeatPlan.p1_uniform(1, 15, 4)
    L = torch.ones((1, 15), dtype=torch.float64, device="cuda")
    R = torch.ones((1, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(stk.ArgumentError, match="fixed_iters"):
        p2.rksm(L, R, fixed_iters=-1)
    with pytest.raises(stk.ArgumentError, match="rank"):
        p2.solve_factored(torch.ones((17, 15), dtype=torch.float64, device="cuda"),
                          torch.ones((17, 4), dtype=torch.float64, device="cuda"))


@pytest.mark.gpu
def test_wave_plan_errors(stk, cuda):
    import torch
    sm = stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, 8))
    tm = stk.wave_time_matrices(stk.TimeGrid(8, 1.0))
    plan = stk.WavePlan(sm, tm, precond=False)
    b = torch.ones(plan.N, dtype=torch.float64, device="cuda")
    with pytest.raises(stk.ArgumentError, match="eigenpairs|precond"):
        plan.two_term_solve(b)
    with pytest.raises(stk.ArgumentError, match="precond"):
        plan.gmres(b, stk.GmresConfig(tol=1e-8, maxit=5))
    with pytest.raises(stk.ArgumentError, match="length"):
        plan.apply(torch.ones(plan.N + 1, dtype=torch.float64, device="cuda"))
    # TwoTermPrecond's solvability check (stk/sylvester.hpp:158-160)
    bad = stk.EigPair(-np.ones(sm.M.n) * 1e9, np.eye(sm.M.n))
    with pytest.raises(stk.SolvabilityError, match="not solvable"):
        stk.WavePlan(sm, tm, space_eig=bad)
