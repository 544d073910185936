"""LuDirect on the device (gadi_lu.cu) against the reference's BandLU.

BandLU (band_lu.cpp:60-172) is the reference's default inner method
(inner_solver.hpp:21). The device factors H and S in u_r with the reference's
per-op rounding and element-wise operation order, so factors, inner solutions
and whole solves are bit for bit the reference's (golden vectors from the
reference itself, tests/golden) and the pinned oracle's. Residual histories
carry the binary64 norm2_64 summation-order tolerance of test_gpu_parity.py.
"""
import os

import numpy as np
import pytest

import paper_2501_04229_b200 as g
from oracle import CSR, DOUBLE, HALF, SINGLE, Config

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz")
PREC = {"h": HALF, "s": SINGLE, "d": DOUBLE}
HIST_RTOL = 1e-13
LU = g.InnerSolverSpec(g.InnerMethod.LuDirect, 1e-2, 1000, 30)


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)


def same(a, b):
    return np.array_equal(bits(a), bits(b))


def systems(orc, n, r=None):
    S = g.build_convdiff3d(n, r=r)
    A = orc.convdiff(n, S.t1, S.t2, S.t3)
    return A, [g.CudaGadiSystem(S), g.CudaGadiSystem(g.SparseMatrix(A.n, A.n, A.rp, A.ci, A.v))]


@pytest.mark.parametrize("n", [5, 8])
@pytest.mark.parametrize("p", ["h", "s", "d"])
def test_lu_inner_golden(orc, gold, n, p):
    """solve_H / solve_S of the reference's convdiff (beta = 1) at alpha = 0.5
    equal the reference's BandLU solves (golden vectors)."""
    A, syss = systems(orc, n)
    for sysx in syss:
        sysx.prepare(0.5, 1.0, g.Precision(PREC[p]), LU)
        for which, f in (("H", sysx.solve_H), ("S", sysx.solve_S)):
            x, it, st = f(gold[f"lu_k{n}{which}_{p}_rhs"])
            assert it == 0 and st == g.InnerStatus.Converged
            assert same(x, gold[f"lu_k{n}{which}_{p}_x"]), (n, p, which)


@pytest.mark.parametrize("p", ["h", "s", "d"])
def test_lu_pivoting_golden(orc, gold, p):
    """Strong convection (r = 0.45) and alpha = 0.02: S is far from diagonally
    dominant, so the elimination swaps rows (in and beyond each 32-step block
    of the solves)."""
    A, syss = systems(orc, 6, r=0.45)
    for sysx in syss:
        sysx.prepare(0.02, 1.0, g.Precision(PREC[p]), LU)
        for which, f in (("H", sysx.solve_H), ("S", sysx.solve_S)):
            x, _, st = f(gold[f"lu_piv{which}_{p}_rhs"])
            assert st == g.InnerStatus.Converged
            assert same(x, gold[f"lu_piv{which}_{p}_x"]), (p, which)


@pytest.mark.parametrize("n,r,alpha", [(16, None, 0.1), (12, 0.45, 0.01), (16, 0.3, 0.05)])
@pytest.mark.parametrize("fmt", [HALF, SINGLE, DOUBLE])
def test_lu_inner_vs_oracle(orc, n, r, alpha, fmt):
    """Larger bands (kl = n^2 = 256 > one 32-column panel of the factorization
    and one 32-step block of the solves) against the pinned oracle."""
    A, syss = systems(orc, n, r)
    H, S = orc.regularize(A, alpha)
    rng = np.random.default_rng(n)
    for sysx in syss:
        sysx.prepare(alpha, 1.0, g.Precision(fmt), LU)
        for M, f in ((H, sysx.solve_H), (S, sysx.solve_S)):
            rhs = orc.round(rng.uniform(-1, 1, A.n), fmt)
            want, st = orc.lu_solve(M, rhs, fmt)
            x, _, dst = f(rhs)
            assert st == 0 and dst == g.InnerStatus.Converged
            assert same(x, want)


@pytest.mark.parametrize("fmt", [HALF, SINGLE, DOUBLE])
def test_lu_band_csr_vs_oracle(orc, fmt):
    """A general CSR (BASELINE configs[3] family, small): random band of
    +-150 columns, bandwidths from the union pattern."""
    A = orc.band(3000, k_off=8, band=150, seed=5)
    alpha = 0.3
    H, S = orc.regularize(A, alpha)
    sysx = g.CudaGadiSystem(g.SparseMatrix(A.n, A.n, A.rp, A.ci, A.v))
    sysx.prepare(alpha, 1.0, g.Precision(fmt), LU)
    rng = np.random.default_rng(3)
    for M, f in ((H, sysx.solve_H), (S, sysx.solve_S)):
        rhs = orc.round(rng.uniform(-1, 1, A.n), fmt)
        want, st = orc.lu_solve(M, rhs, fmt)
        x, _, _ = f(rhs)
        assert st == 0 and same(x, want)


@pytest.mark.parametrize("tag", ["luh8", "lus8", "lud6", "luh12"])
def test_solve_lu_direct_golden(orc, gold, tag):
    """Whole GADI-IR solves with inner lu_direct = the reference's own runs."""
    n, ur, alpha = gold[f"solve_{tag}_cfg"][:3]
    b = gold[f"solve_{tag}_b"]
    cfg = g.GadiConfig(alpha=float(alpha), xi=1e-20 if int(ur) != HALF else 1e-8, u_r=g.Precision(int(ur)),
                       inner=LU)
    A, _ = systems(orc, int(n))
    info = list(gold[f"solve_{tag}_info"])
    for M in (g.build_convdiff3d(int(n)), g.SparseMatrix(A.n, A.n, A.rp, A.ci, A.v)):
        res = g.gadi_ir_solve(M, b, g.hss_split(M), cfg)
        rep = res.report
        assert [int(rep.status), rep.outer_iters, rep.inner_iter_totals, rep.inner_stagnations] == info
        assert same(res.x, gold[f"solve_{tag}_x"])
        assert np.allclose(rep.rel_residual_history, gold[f"solve_{tag}_hist"], rtol=HIST_RTOL, atol=0)


def test_lu_singular_and_overflow(orc):
    """prepare's exceptions (band_lu.cpp:106-108, 132-134): GADI_E_SINGULAR /
    GADI_E_OVERFLOW from gadi_cuda_prepare, SingularInPrecision /
    OverflowDetected statuses from the solve (solver.cpp:74-82), as the oracle."""
    z = g.SparseMatrix(3, 3, [0, 1, 2, 3], [0, 1, 2], [0.0, 0.0, 0.0])  # H = alpha I
    big = g.SparseMatrix(3, 3, [0, 1, 2, 3], [0, 1, 2], [70000.0, 1.0, 2.0])  # rounds to inf in binary16
    b = np.array([1.0, -2.0, 0.5])
    for M, alpha, st, exc in ((z, 1e-6, g.SolveStatus.SingularInPrecision, g.SingularInPrecision),
                              (big, 0.5, g.SolveStatus.OverflowDetected, g.OverflowDetected)):
        sysx = g.CudaGadiSystem(M, b)
        with pytest.raises(exc):
            sysx.prepare(alpha, 1.0, g.Precision.Half, LU)
        cfg = g.GadiConfig(alpha=alpha, u_r=g.Precision.Half, inner=LU)
        res = g.gadi_ir_solve(M, b, g.hss_split(M), cfg)
        _, wrep, _ = orc.solve(CSR(3, M.row_ptr, M.col_idx, M.values), b,
                               Config.make(alpha=alpha, u_r=HALF, method=0))
        assert res.report.status == st == wrep.status and res.report.outer_iters == 0


def test_lu_single_precision_accum_ignored(orc):
    """LuDirect rounds every op to u_r whatever `accum` says (the reference LU)."""
    A, syss = systems(orc, 8)
    H, _ = orc.regularize(A, 0.2)
    rhs = orc.round(np.random.default_rng(1).uniform(-1, 1, A.n), HALF)
    want, _ = orc.lu_solve(H, rhs, HALF)
    sysx = syss[0]
    sysx.prepare(0.2, 1.0, g.Precision.Half, LU, g.Accum.Fp32)
    x, _, _ = sysx.solve_H(rhs)
    assert same(x, want)
