"""The reference's own solver/inner-solver test assertions, re-expressed.

Source: /root/reference/proj/tests/test_solver.cpp and test_inner_solver.cpp
(doctest; the cited line is on each test). Each case runs twice: on the CPU
oracle (always) and on the device path through the C ABI (-m gpu). The
reference runs most of them with its default band-LU inner solver
(inner_solver.hpp:21), which has no device implementation; here the inner
method is CG (GMRES on S, solver.cpp:217-221) with a tight epsilon, which the
reference's own "krylov inner solves drive the outer loop" case
(test_solver.cpp:185-203) also uses.
"""
import numpy as np
import pytest

import paper_2501_04229_b200 as g
from oracle import CSR, CG, DOUBLE, GMRES, HALF, SINGLE, Config, Oracle

ORC = Oracle()


def csr_identity(n):
    return CSR(n, np.arange(n + 1), np.arange(n), np.ones(n))


def csr_diag(d):
    n = len(d)
    return CSR(n, np.arange(n + 1), np.arange(n), np.asarray(d, np.float64))


KRYLOV = dict(method=CG, tol_epsilon=1e-12, max_inner_iters=200)
# the reference's tests run its default InnerSolverSpec{} (lu_direct, inner_solver.hpp:20-25)
LU = dict(method=0, tol_epsilon=1e-2, max_inner_iters=1000)


class OracleBackend:
    name = "oracle"

    def __init__(self, inner=KRYLOV):
        self.inner = inner

    def solve(self, A, b, stencil_n=None, x0=None, **kw):
        cfg = Config.make(**{**self.inner, **kw})
        try:
            x, rep, hist = ORC.solve(A, b, cfg, x0=x0)
        except ValueError as e:
            raise g.ParameterError(str(e))
        return x, g.SolveStatus(rep.status), rep.outer_iters, hist, rep.inner_iter_totals, rep.final_rres

    def krylov(self, A, which, rhs, method, eps, max_inner, restart, fmt, stop, alpha):
        H, S = ORC.regularize(A, alpha)
        x, it, st = ORC.krylov(H if which == "H" else S, rhs, method, eps, max_inner, restart, fmt, stop)
        return x, it, g.InnerStatus(st)


class DeviceBackend:
    name = "device"

    def __init__(self, inner=KRYLOV):
        self.inner = inner

    def _cfg(self, kw):
        kw = {**self.inner, **kw}
        inner = g.InnerSolverSpec(g.InnerMethod(kw.pop("method")), kw.pop("tol_epsilon"), kw.pop("max_inner_iters"),
                                  kw.pop("restart", 30))
        for k in ("u_r", "u", "u_f"):
            if k in kw:
                kw[k] = g.Precision(kw[k])
        return g.GadiConfig(inner=inner, **kw)

    def solve(self, A, b, stencil_n=None, x0=None, **kw):
        M = g.build_convdiff3d(stencil_n) if stencil_n else g.SparseMatrix(A.n, A.n, A.rp, A.ci, A.v)
        res = g.gadi_ir_solve(M, b, g.hss_split(M), self._cfg(kw), x0=x0)
        r = res.report
        return res.x, r.status, r.outer_iters, r.rel_residual_history, r.inner_iter_totals, r.final_rres

    def krylov(self, A, which, rhs, method, eps, max_inner, restart, fmt, stop, alpha):
        s = g.CudaGadiSystem(g.SparseMatrix(A.n, A.n, A.rp, A.ci, A.v))
        s.prepare(alpha, 1.0, g.Precision(fmt), g.InnerSolverSpec(g.InnerMethod(method), eps, max_inner, restart))
        s.set_inner_stop_norm(stop)
        x, it, st = s.solve_H(rhs) if which == "H" else s.solve_S(rhs)
        s.close()
        return x, it, st


@pytest.fixture(params=["oracle-krylov", "oracle-lu", pytest.param("device-krylov", marks=pytest.mark.gpu),
                        pytest.param("device-lu", marks=pytest.mark.gpu)])
def be(request):
    where, inner = request.param.split("-")
    inner = LU if inner == "lu" else KRYLOV
    return OracleBackend(inner) if where == "oracle" else DeviceBackend(inner)


def convdiff(n):
    return ORC.convdiff(n), ORC.matvec(ORC.convdiff(n), np.ones(n ** 3), DOUBLE)


@pytest.mark.parametrize("prec", [(DOUBLE, DOUBLE, DOUBLE), (HALF, DOUBLE, DOUBLE), (HALF, SINGLE, SINGLE)])
def test_identity_two_outer_iterations(be, prec):
    """test_solver.cpp:13-31: A = I, alpha = 1, xi = 0.1 -> <= 2 outer iterations."""
    A = csr_identity(6)
    b = np.array([1.0, -2.0, 3.0, 0.5, 0.0, 4.0])
    ur, u, uf = prec
    _, st, outer, *_ = be.solve(A, b, alpha=1.0, omega=1.0, xi=0.1, u_r=ur, u=u, u_f=uf)
    assert st == g.SolveStatus.Converged and outer <= 2


def test_report_invariants(be):
    """test_solver.cpp:33-52: history shape, converged tolerance, monotone tail, A x = b."""
    A, b = convdiff(4)
    x, st, outer, hist, _, final = be.solve(A, b, stencil_n=4, alpha=0.5, xi=1e-20)
    assert st == g.SolveStatus.Converged
    assert len(hist) == outer + 1 and hist[0] == 1.0 and final == hist[-1] and final * final <= 1e-20
    assert len(hist) >= 5 and all(hist[i + 1] <= hist[i] for i in range(len(hist) - 5, len(hist) - 1))
    r = ORC.residual(A, x, b, DOUBLE, DOUBLE)
    assert ORC.norm2_64(r) / ORC.norm2_64(b) <= 1e-9


def test_exact_start_zero_iterations(be):
    """test_solver.cpp:54-66: x0 = x* converges in zero outer iterations."""
    A, b = convdiff(3)
    _, st, outer, *_ = be.solve(A, b, stencil_n=3, x0=np.ones(27), alpha=1.0)
    assert st == g.SolveStatus.Converged and outer == 0


def test_overflow_detected(be):
    """test_solver.cpp:146-160: x* = 7e4 overflows binary16 in the u = half update."""
    A = csr_diag([0.001] * 3)
    b = np.full(3, 70.0)
    _, st, outer, hist, *_ = be.solve(A, b, alpha=0.001, u_r=HALF, u=HALF, u_f=HALF, xi=1e-4, max_outer_iters=4000)
    assert st == g.SolveStatus.OverflowDetected
    assert len(hist) == outer + 1


def test_max_iters(be):
    """test_solver.cpp:161-170: the outer cap is reported as MaxIters."""
    A, b = convdiff(3)
    _, st, outer, *_ = be.solve(A, b, stencil_n=3, alpha=0.01, xi=1e-26, max_outer_iters=5)
    assert st == g.SolveStatus.MaxIters and outer == 5


def test_stall_window(be):
    """test_solver.cpp:172-182: half floor without residual scaling -> Stalled."""
    A, b = convdiff(3)
    _, st, _, _, _, final = be.solve(A, b, stencil_n=3, alpha=10.0, u_r=HALF, xi=1e-26, stall_window=200,
                                     max_outer_iters=20000, residual_scaling=0)
    assert st == g.SolveStatus.Stalled and final > 1e-13


def test_krylov_drives_outer_below_target(be):
    """test_solver.cpp:185-203."""
    A, b = convdiff(4)
    _, st, _, _, inner, final = be.solve(A, b, stencil_n=4, alpha=0.5, xi=1e-18, method=CG, tol_epsilon=1e-12,
                                         max_inner_iters=3000, max_outer_iters=10000)
    assert st == g.SolveStatus.Converged and final <= 1e-9 and inner > 0


def test_bitwise_determinism(be):
    """test_solver.cpp:205-219: two identical solves agree bit for bit."""
    A, b = convdiff(5)
    kw = dict(stencil_n=5, alpha=0.5, u_r=HALF, xi=1e-20, stall_window=300, residual_scaling=0,
              max_inner_iters=30)
    x1, _, o1, h1, *_ = be.solve(A, b, **kw)
    x2, _, o2, h2, *_ = be.solve(A, b, **kw)
    assert o1 == o2 and np.array_equal(x1.view(np.int64), x2.view(np.int64))
    assert np.array_equal(np.asarray(h1).view(np.int64), np.asarray(h2).view(np.int64))


@pytest.mark.parametrize("bad", [dict(alpha=-1.0), dict(omega=2.0), dict(u=HALF, u_f=DOUBLE, u_r=DOUBLE)])
def test_config_validation(be, bad):
    """test_solver.cpp:221-235: parameter errors throw ParameterError."""
    A, b = convdiff(2)
    with pytest.raises(g.ParameterError):
        be.solve(A, b, stencil_n=2, **bad)


def test_limiting_accuracy(be):
    """test_solver.cpp:237-260: the floor follows u, the rate follows u_r."""
    A, b = convdiff(6)
    kw = dict(stencil_n=6, alpha=10.0, max_outer_iters=20000, stall_window=400)
    hdd = be.solve(A, b, u_r=HALF, u=DOUBLE, u_f=DOUBLE, xi=1e-20, **kw)
    sdd = be.solve(A, b, u_r=SINGLE, u=DOUBLE, u_f=DOUBLE, xi=1e-20, **kw)
    sss = be.solve(A, b, u_r=SINGLE, u=SINGLE, u_f=SINGLE, xi=1e-8, **kw)
    assert hdd[1] == g.SolveStatus.Converged and sdd[1] == g.SolveStatus.Converged
    assert sss[5] >= 1e4 * hdd[5] and sss[5] >= 1e4 * sdd[5]


def test_cg_identity_one_iteration(be):
    """test_inner_solver.cpp:152-160: CG on I converges in <= 1 iteration."""
    A = csr_identity(3)
    rhs = np.array([1.0, -2.0, 0.5])
    # H = alpha I + M with M = I (hss of I); alpha -> tiny so H ~ I
    x, it, st = be.krylov(A, "H", rhs, CG, 1e-10, 1000, 30, DOUBLE, np.linalg.norm(rhs), 1e-300)
    assert st == g.InnerStatus.Converged and it <= 1
    np.testing.assert_allclose(x, rhs, rtol=1e-9)


def test_cg_half_on_convdiff_H(be):
    """test_inner_solver.cpp:162-176: CG in half on H (n = 8, alpha = 0.5) to 1e-2."""
    A = ORC.convdiff(8)
    rng = np.random.default_rng(123)
    r = ORC.round(rng.uniform(-1, 1, 512), HALF)
    x, it, st = be.krylov(A, "H", r, CG, 1e-2, 512, 30, HALF, ORC.norm2_64(r), 0.5)
    H, _ = ORC.regularize(A, 0.5)
    res = ORC.norm2_64(ORC.residual(H, x, r, DOUBLE, DOUBLE))
    assert st == g.InnerStatus.Converged and it <= 512 and res <= 2e-2 * ORC.norm2_64(r) + 1e-3


def test_gmres_on_S_and_stagnation(be):
    """test_inner_solver.cpp:179-214."""
    A = ORC.convdiff(4)
    r = np.ones(64)
    x, it, st = be.krylov(A, "S", r, GMRES, 1e-6, 500, 30, DOUBLE, ORC.norm2_64(r), 0.5)
    _, S = ORC.regularize(A, 0.5)
    assert st == g.InnerStatus.Converged
    assert ORC.norm2_64(ORC.residual(S, x, r, DOUBLE, DOUBLE)) <= 1e-5 * ORC.norm2_64(r)
    _, _, st2 = be.krylov(A, "S", r, GMRES, 1e-14, 2, 30, DOUBLE, ORC.norm2_64(r), 0.5)
    assert st2 == g.InnerStatus.Stagnated
    A8 = ORC.convdiff(8)
    rng = np.random.default_rng(5)
    rr = ORC.round(rng.uniform(-1, 1, 512), HALF)
    _, _, st3 = be.krylov(A8, "S", rr, GMRES, 1e-3, 300, 30, HALF, ORC.norm2_64(rr), 0.01)
    assert st3 != g.InnerStatus.Converged
