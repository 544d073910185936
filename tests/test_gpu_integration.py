"""The reference's own outer loop driving the device: run_gadi_ir
(solver.cpp:57-179, compiled from /root/reference into oracle/_ref) over a
CudaGadiSystem whose virtuals are the C ABI (oracle/ref_cuda_adapter.cpp,
the binding INTEGRATION.md describes). Its result must equal the
device-resident loop's and the oracle's bit for bit."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2501_04229_b200 as g
from oracle import CG, HALF, LU_DIRECT, SINGLE, Config, Report

pytestmark = pytest.mark.gpu
LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "libgadi_ref_cuda.so")


@pytest.fixture(scope="module")
def adapter():
    if not os.path.exists(LIB):
        pytest.skip("oracle/_ref/libgadi_ref_cuda.so not built (needs /root/reference at build time)")
    g.lib()
    L = C.CDLL(LIB)
    f64p = C.POINTER(C.c_double)
    L.refcuda_solve_stencil.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double, f64p, C.POINTER(Config),
                                        f64p, f64p, C.c_int, C.POINTER(Report)]
    return L


@pytest.mark.parametrize("n,ur,alpha,method", [(16, SINGLE, 0.1, CG), (8, HALF, 0.5, CG), (8, HALF, 0.3, LU_DIRECT),
                                               (6, SINGLE, 0.5, LU_DIRECT)])
def test_reference_loop_over_device_system(orc, adapter, n, ur, alpha, method):
    S = g.build_convdiff3d(n)
    A = orc.convdiff(n, S.t1, S.t2, S.t3)
    _, b = orc.make_rhs(A, 0, 0.0, 1.0)
    cfg = Config.make(alpha=alpha, xi=1e-20, u_r=ur, method=method, tol_epsilon=1e-12, max_inner_iters=50)
    x = np.zeros(A.n)
    hist = np.zeros(10000)
    rep = Report()
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    rc = adapter.refcuda_solve_stencil(n, S.t1, S.t2, S.t3, p(b), C.byref(cfg), p(x), p(hist), 10000,
                                       C.byref(rep))
    assert rc == 0
    wx, wrep, _ = orc.solve(A, b, cfg)
    res = g.gadi_ir_solve(S, b, g.hss_split(S), g.GadiConfig(
        alpha=alpha, xi=1e-20, u_r=g.Precision(ur), inner=g.InnerSolverSpec(g.InnerMethod(method), 1e-12, 50, 30)))
    assert rep.status == wrep.status == int(res.report.status)
    assert rep.outer_iters == wrep.outer_iters == res.report.outer_iters
    assert np.array_equal(x.view(np.int64), wx.view(np.int64))
    assert np.array_equal(res.x.view(np.int64), wx.view(np.int64))
