"""Parity of the sm_100a path (through the C ABI) against the CPU oracle.

The oracle (oracle/gadi_oracle.c) is pinned bit for bit to the reference in
test_oracle_pin.py. Integer/byte-exact claims here are bitwise: the device
reproduces the reference's per-op rounding (kernels.cpp:26-54) and its
pairwise-sum tree (kernels.cpp:33-39), so binary64/32/16-native kernels and
whole solves agree to the last bit; binary64 norms (norm2_64,
kernels.cpp:184-194) are summed in a different order and agree to 1e-14
relative, which is the tolerance written below for residual histories.
"""
import numpy as np
import pytest

import paper_2501_04229_b200 as g
from oracle import CG, GMRES, DOUBLE, HALF, SINGLE, Config

pytestmark = pytest.mark.gpu

HIST_RTOL = 1e-13  # binary64 norm summation order (norm2_64) only


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)


def same(a, b):
    return np.array_equal(bits(a), bits(b))


def stencil_and_csr(orc, n, r=None):
    S = g.build_convdiff3d(n, r=r)
    A = orc.convdiff(n, S.t1, S.t2, S.t3)
    return S, A


@pytest.mark.parametrize("n", [2, 3, 5, 8, 16])
def test_apply_A_bitwise(orc, n):
    S, A = stencil_and_csr(orc, n)
    x = np.random.default_rng(n).uniform(-1, 1, A.n)
    sysS = g.CudaGadiSystem(S)
    sysC = g.CudaGadiSystem(g.SparseMatrix(A.n, A.n, A.rp, A.ci, A.v))
    want = orc.matvec(A, x, DOUBLE)
    assert same(sysS.apply("A", x), want)
    assert same(sysC.apply("A", x), want)


@pytest.mark.parametrize("n", [3, 8, 16])
@pytest.mark.parametrize("uf", [HALF, SINGLE, DOUBLE])
def test_residual_uf_bitwise(orc, n, uf):
    S, A = stencil_and_csr(orc, n)
    rng = np.random.default_rng(7 + n)
    x = orc.round(rng.uniform(-1, 1, A.n), uf)
    b = rng.uniform(-3, 3, A.n)
    sysS = g.CudaGadiSystem(S, b)
    want = orc.residual(A, x, b, uf, DOUBLE)
    assert same(sysS.residual_uf(x, g.Precision(uf)), want)
    t = orc.norm2_64(orc.residual(A, x, b, DOUBLE, DOUBLE))
    assert abs(sysS.true_residual_norm(x) - t) <= 1e-14 * t


@pytest.mark.parametrize("n", [3, 5, 8, 16])
@pytest.mark.parametrize("fmt", [HALF, SINGLE, DOUBLE])
def test_apply_H_S_bitwise(orc, n, fmt):
    S, A = stencil_and_csr(orc, n)
    alpha = 0.1
    H, Sm = orc.regularize(A, alpha)
    x = orc.round(np.random.default_rng(n).uniform(-1, 1, A.n), fmt)
    for sysx in (g.CudaGadiSystem(S), g.CudaGadiSystem(g.SparseMatrix(A.n, A.n, A.rp, A.ci, A.v))):
        sysx.prepare(alpha, 1.0, g.Precision(fmt), g.InnerSolverSpec(g.InnerMethod.Cg, 1e-6, 10, 30))
        for name, M in (("H", H), ("S", Sm)):
            Mr = type(M)(M.n, M.rp, M.ci, orc.round(M.v, fmt))
            assert same(sysx.apply(name, x), orc.matvec(Mr, x, fmt)), (name, fmt)


@pytest.mark.parametrize("n", [3, 4, 5, 8, 16])
@pytest.mark.parametrize("fmt", [HALF, SINGLE, DOUBLE])
@pytest.mark.parametrize("method", [CG, GMRES])
def test_krylov_bitwise(orc, n, fmt, method):
    S, A = stencil_and_csr(orc, n)
    alpha = 0.5
    H, Sm = orc.regularize(A, alpha)
    rhs = orc.round(np.random.default_rng(3 * n + fmt).uniform(-1, 1, A.n), fmt)
    stop = orc.norm2_64(rhs)
    eps, max_inner, restart = 1e-6, 60, 10
    sysx = g.CudaGadiSystem(S)
    sysx.prepare(alpha, 1.0, g.Precision(fmt), g.InnerSolverSpec(g.InnerMethod(method), eps, max_inner, restart))
    sysx.set_inner_stop_norm(stop)
    if method == CG:
        x, it, st = sysx.solve_H(rhs)
        wx, wit, wst = orc.krylov(H, rhs, CG, eps, max_inner, restart, fmt, stop)
    else:
        x, it, st = sysx.solve_S(rhs)
        wx, wit, wst = orc.krylov(Sm, rhs, GMRES, eps, max_inner, restart, fmt, stop)
    assert (it, int(st)) == (wit, wst)
    assert same(x, wx)


@pytest.mark.parametrize("n,fmt,alpha", [(8, DOUBLE, 0.5), (8, SINGLE, 0.1), (16, SINGLE, 0.1),
                                         (8, HALF, 0.5), (16, HALF, 0.1), (5, SINGLE, 0.3)])
def test_solve_matches_oracle(orc, n, fmt, alpha):
    """gadi_ir_solve parity: same outer count, same x bit for bit."""
    S, A = stencil_and_csr(orc, n)
    xt, b = orc.make_rhs(A, 0, 0.0, 1.0)
    cfg = Config.make(alpha=alpha, xi=1e-20, u_r=fmt, method=CG, tol_epsilon=1e-12, max_inner_iters=50,
                      stall_window=400)
    wx, wrep, whist = orc.solve(A, b, cfg)
    gcfg = g.GadiConfig(alpha=alpha, xi=1e-20, u_r=g.Precision(fmt),
                        inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 50, 30), stall_window=400)
    res = g.gadi_ir_solve(S, b, g.hss_split(S), gcfg)
    assert int(res.report.status) == wrep.status
    assert res.report.outer_iters == wrep.outer_iters
    assert res.report.inner_iter_totals == wrep.inner_iter_totals
    assert same(res.x, wx)
    np.testing.assert_allclose(res.report.rel_residual_history, whist, rtol=HIST_RTOL, atol=0)


def test_solve_csr_matches_oracle(orc):
    n = 8
    S, A = stencil_and_csr(orc, n)
    xt, b = orc.make_rhs(A, 1, -1.0, 1.0)
    cfg = Config.make(alpha=0.2, xi=1e-20, u_r=SINGLE, method=CG, tol_epsilon=1e-12, max_inner_iters=50)
    wx, wrep, _ = orc.solve(A, b, cfg)
    Ag = g.SparseMatrix(A.n, A.n, A.rp, A.ci, A.v)
    gcfg = g.GadiConfig(alpha=0.2, xi=1e-20, u_r=g.Precision.Single,
                        inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 50, 30))
    res = g.gadi_ir_solve(Ag, b, g.hss_split(Ag), gcfg)
    assert res.report.outer_iters == wrep.outer_iters
    assert same(res.x, wx)


@pytest.mark.parametrize("n", [1, 2, 3, 7, 64, 100, 1000, 4096, 65536, 100003])
@pytest.mark.parametrize("p", [HALF, SINGLE, DOUBLE])
def test_device_dot_norm2_bitwise(orc, n, p):
    rng = np.random.default_rng(n)
    x = orc.round(rng.uniform(-1, 1, n), p)
    y = orc.round(rng.uniform(-1, 1, n), p)
    assert same([g.device_dot(x, y, g.Precision(p))], [orc.dot(x, y, p)])
    assert same([g.device_norm2(x, g.Precision(p))], [orc.norm2(x, p)])


# ---- the device path against the reference's own outputs (tests/golden) ----
GOLD = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "reference_vectors.npz")
PREC = {"h": HALF, "s": SINGLE, "d": DOUBLE}


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.mark.parametrize("n", [5, 8])
@pytest.mark.parametrize("p", ["h", "s", "d"])
@pytest.mark.parametrize("meth", ["cg", "gm"])
def test_golden_krylov(gold, n, p, meth):
    sysx = g.CudaGadiSystem(g.build_convdiff3d(n))
    sysx.prepare(0.5, 1.0, g.Precision(PREC[p]),
                 g.InnerSolverSpec(g.InnerMethod.Cg if meth == "cg" else g.InnerMethod.Gmres, 1e-6, 60, 10))
    rhs = gold[f"k{n}_rhs_{p}"]
    from oracle import Oracle
    sysx.set_inner_stop_norm(Oracle().norm2_64(rhs))
    x, it, st = sysx.solve_H(rhs) if meth == "cg" else sysx.solve_S(rhs)
    assert [it, int(st)] == list(gold[f"k{n}_{meth}_{p}_info"])
    assert same(x, gold[f"k{n}_{meth}_{p}_x"])


@pytest.mark.parametrize("tag", ["s16", "h16", "d8", "s8b"])
def test_golden_solve(gold, tag):
    n, ur, alpha, seed, lo, hi = gold[f"solve_{tag}_cfg"]
    S = g.build_convdiff3d(int(n))
    cfg = g.GadiConfig(alpha=alpha, xi=1e-20, u_r=g.Precision(int(ur)),
                       inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 50, 30))
    res = g.gadi_ir_solve(S, gold[f"solve_{tag}_b"], g.hss_split(S), cfg)
    info = gold[f"solve_{tag}_info"]
    assert [int(res.report.status), res.report.outer_iters, res.report.inner_iter_totals,
            res.report.inner_stagnations] == list(info)
    assert same(res.x, gold[f"solve_{tag}_x"])
    np.testing.assert_allclose(res.report.rel_residual_history, gold[f"solve_{tag}_hist"], rtol=HIST_RTOL, atol=0)


# ---- BASELINE configs[3] family: device generator, device HSS split, SELL kernels ----
@pytest.mark.parametrize("N,k,band", [(4096, 26, 256), (1000, 8, 40)])
def test_band_generator_split_and_solve(orc, N, k, band):
    A = orc.band(N, k, band, 2)
    Bg = g.build_band_csr(N, k, band, 2)
    s = g.CudaGadiSystem(Bg)
    x = np.random.default_rng(N).uniform(-1, 1, N)
    assert same(s.apply("A", x), orc.matvec(A, x, DOUBLE))  # generator + SELL(A), bit for bit
    H, S = orc.regularize(A, 0.7)
    s.prepare(0.7, 1.0, g.Precision.Single, g.InnerSolverSpec(g.InnerMethod.Cg, 1e-6, 10, 30))
    xs = orc.round(x, SINGLE)
    for name, M in (("H", H), ("S", S)):  # device split + SELL(H, S)
        Mr = type(M)(M.n, M.rp, M.ci, orc.round(M.v, SINGLE))
        assert same(s.apply(name, xs), orc.matvec(Mr, xs, SINGLE)), name
    s.close()
    _, b = orc.make_rhs(A, 1, -1.0, 1.0)
    cfg = Config.make(alpha=2.0, xi=1e-20, u_r=SINGLE, method=CG, tol_epsilon=1e-12, max_inner_iters=20)
    wx, wrep, _ = orc.solve(A, b, cfg)
    res = g.gadi_ir_solve(Bg, b, g.hss_split(Bg), g.GadiConfig(
        alpha=2.0, xi=1e-20, u_r=g.Precision.Single, inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 20, 30)))
    assert int(res.report.status) == wrep.status == 0
    assert res.report.outer_iters == wrep.outer_iters
    assert same(res.x, wx)


@pytest.mark.parametrize("fmt", [HALF, SINGLE, DOUBLE])
@pytest.mark.parametrize("method", [CG, GMRES])
def test_band_krylov_bitwise(orc, fmt, method):
    """SELL kernels with the shared-memory operand window (N = 2^13, band 300)
    against the oracle's Krylov solvers; the right-hand side carries +-0 entries
    so the GMRES residual from x = 0 exercises the zflag shortcut."""
    N, k, band, alpha = 8192, 26, 300, 3.0
    A = orc.band(N, k, band, 3)
    H, Sm = orc.regularize(A, alpha)
    rhs = orc.round(np.random.default_rng(fmt).uniform(-1, 1, N), fmt)
    rhs[::7] = 0.0
    rhs[3::7] = -0.0
    stop = orc.norm2_64(rhs)
    eps, max_inner, restart = 1e-8, 40, 12
    s = g.CudaGadiSystem(g.build_band_csr(N, k, band, 3))
    s.prepare(alpha, 1.0, g.Precision(fmt), g.InnerSolverSpec(g.InnerMethod(method), eps, max_inner, restart))
    s.set_inner_stop_norm(stop)
    x, it, st = s.solve_H(rhs) if method == CG else s.solve_S(rhs)
    wx, wit, wst = orc.krylov(H if method == CG else Sm, rhs, method, eps, max_inner, restart, fmt, stop)
    assert (it, int(st)) == (wit, wst)
    assert same(x, wx)


@pytest.mark.parametrize("n,fmt", [(8, HALF), (8, SINGLE), (5, DOUBLE), (16, HALF)])
def test_gmres_zero_start_signed_zeros(orc, n, fmt):
    """r = rhs - S*0 keeps -0 only in rows whose stored coefficients are all
    sign-clear (the reference's fold; gadi_kernels.cuh zero_resid)."""
    S, A = stencil_and_csr(orc, n)
    alpha = 0.5
    _, Sm = orc.regularize(A, alpha)
    rhs = orc.round(np.random.default_rng(n + fmt).uniform(-1, 1, A.n), fmt)
    rhs[::3] = -0.0
    rhs[1::5] = 0.0
    stop = orc.norm2_64(rhs)
    sysx = g.CudaGadiSystem(S)
    sysx.prepare(alpha, 1.0, g.Precision(fmt), g.InnerSolverSpec(g.InnerMethod.Gmres, 1e-6, 30, 7))
    sysx.set_inner_stop_norm(stop)
    x, it, st = sysx.solve_S(rhs)
    wx, wit, wst = orc.krylov(Sm, rhs, GMRES, 1e-6, 30, 7, fmt, stop)
    assert (it, int(st)) == (wit, wst)
    assert same(x, wx)


@pytest.mark.parametrize("sparse", [False, True])
def test_gmres_overflowed_coefficients(orc, sparse):
    """alpha beyond binary16 range: S's diagonal rounds to inf, the residual
    from x = 0 is NaN in those rows, GMRES reports Overflow like the reference."""
    n, alpha = 8, 1e5
    S, A = stencil_and_csr(orc, n)
    _, Sm = orc.regularize(A, alpha)
    rhs = orc.round(np.random.default_rng(1).uniform(-1, 1, A.n), HALF)
    stop = orc.norm2_64(rhs)
    sysx = g.CudaGadiSystem(g.SparseMatrix(A.n, A.n, A.rp, A.ci, A.v) if sparse else S)
    sysx.prepare(alpha, 1.0, g.Precision.Half, g.InnerSolverSpec(g.InnerMethod.Gmres, 1e-6, 30, 7))
    sysx.set_inner_stop_norm(stop)
    x, it, st = sysx.solve_S(rhs)
    wx, wit, wst = orc.krylov(Sm, rhs, GMRES, 1e-6, 30, 7, HALF, stop)
    assert (it, int(st)) == (wit, wst)
    assert int(st) == 2  # Overflow
    assert same(x, wx)


@pytest.mark.parametrize("kind", ["stencil", "band"])
def test_solve_accum_fp32_matches_oracle(orc, kind):
    """binary16 storage with binary32 arithmetic (the C3/C4 inner mode,
    GADI_ACCUM_FP32): whole solves bit for bit against the oracle."""
    if kind == "stencil":
        S, A = stencil_and_csr(orc, 16, r=0.5)
        dev = S
    else:
        A = orc.band(4096, 26, 256, 5)
        dev = g.build_band_csr(4096, 26, 256, 5)
    _, b = orc.make_rhs(A, 1, -1.0, 1.0)
    alpha = 0.4 if kind == "stencil" else 4.0
    cfg = Config.make(alpha=alpha, xi=1e-20, u_r=HALF, method=CG, tol_epsilon=1e-12, max_inner_iters=5,
                      stall_window=400, accum=1)
    wx, wrep, _ = orc.solve(A, b, cfg)
    res = g.gadi_ir_solve(dev, b, g.hss_split(dev), g.GadiConfig(
        alpha=alpha, xi=1e-20, u_r=g.Precision.Half, accum=g.Accum.Fp32, stall_window=400,
        inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 5, 30)))
    assert int(res.report.status) == wrep.status
    assert res.report.outer_iters == wrep.outer_iters
    assert res.report.inner_iter_totals == wrep.inner_iter_totals
    assert same(res.x, wx)


@pytest.mark.parametrize("kind", ["stencil", "band"])
@pytest.mark.parametrize("method", [CG, GMRES])
def test_krylov_accum_fp32_bitwise(orc, kind, method):
    """GADI_ACCUM_FP32 (binary16 storage, binary32 arithmetic): CG / GMRES bit
    for bit against the oracle's restatement of that mode (af = SINGLE)."""
    if kind == "stencil":
        S, A = stencil_and_csr(orc, 16, r=0.3)
        dev = S
    else:
        A = orc.band(8192, 26, 300, 4)
        dev = g.build_band_csr(8192, 26, 300, 4)
    alpha = 0.6 if kind == "stencil" else 3.0
    H, Sm = orc.regularize(A, alpha)
    rhs = orc.round(np.random.default_rng(11).uniform(-1, 1, A.n), HALF)
    rhs[5::9] = -0.0
    stop = orc.norm2_64(rhs)
    eps, max_inner, restart = 1e-9, 40, 12
    sysx = g.CudaGadiSystem(dev)
    sysx.prepare(alpha, 1.0, g.Precision.Half, g.InnerSolverSpec(g.InnerMethod(method), eps, max_inner, restart),
                 g.Accum.Fp32)
    sysx.set_inner_stop_norm(stop)
    x, it, st = sysx.solve_H(rhs) if method == CG else sysx.solve_S(rhs)
    wx, wit, wst = orc.krylov(H if method == CG else Sm, rhs, method, eps, max_inner, restart, HALF, stop,
                              af=SINGLE)
    assert (it, int(st)) == (wit, wst)
    assert same(x, wx)


@pytest.mark.parametrize("n,fmt,accum,alpha", [(16, HALF, True, 0.4), (32, HALF, True, 0.5), (16, SINGLE, False, 0.1),
                                               (8, DOUBLE, False, 0.5)])
def test_speculative_outer_residual_equals_two_pass(orc, monkeypatch, n, fmt, accum, alpha):
    """The single-pass outer residual (s, rhat with the previous step's
    scaling exponent and ||rhat||^2 in one st25 pass, solver.cpp:86-92,
    accepted iff the exponent is unchanged) against the two-pass route
    (residual, then scale/round) forced with GADI_NO_SPEC: identical x,
    residual history and counts, bit for bit, and both equal the oracle."""
    S, A = stencil_and_csr(orc, n, r=0.0975 if n == 32 else None)
    _, b = orc.make_rhs(A, 1, -1.0, 1.0)
    gcfg = g.GadiConfig(alpha=alpha, xi=1e-20, u_r=g.Precision(fmt), stall_window=400,
                        accum=g.Accum.Fp32 if accum else g.Accum.Native,
                        inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 5, 30))
    res = g.gadi_ir_solve(S, b, g.hss_split(S), gcfg)
    monkeypatch.setenv("GADI_NO_SPEC", "1")
    two = g.gadi_ir_solve(S, b, g.hss_split(S), gcfg)
    monkeypatch.delenv("GADI_NO_SPEC")
    assert int(res.report.status) == int(two.report.status) == 0
    assert res.report.outer_iters == two.report.outer_iters
    assert res.report.inner_iter_totals == two.report.inner_iter_totals
    assert same(res.x, two.x)
    assert same(res.report.rel_residual_history, two.report.rel_residual_history)
    cfg = Config.make(alpha=alpha, xi=1e-20, u_r=fmt, method=CG, tol_epsilon=1e-12, max_inner_iters=5,
                      stall_window=400, accum=1 if accum else 0)
    wx, wrep, _ = orc.solve(A, b, cfg)
    assert res.report.outer_iters == wrep.outer_iters
    assert same(res.x, wx)


@pytest.mark.parametrize("method", [CG, GMRES])
def test_fast_binary16_passes_equal_generic_n256(monkeypatch, method):
    """The register-operand binary16 stencil passes (k_st25h: CG p-update +
    SpMV, Arnoldi matvec with the fused v = w/h scale) run
    only when a warp's 32 chunks lie in one grid row (n >= 256); there they
    must equal the generic st25 passes (validated against the oracle at small
    n) bit for bit: GADI_ST25H=0 forces the generic ones."""
    n = 256
    S = g.build_convdiff3d(n, r=0.0975)
    rng = np.random.default_rng(7)
    rhs = rng.uniform(-1, 1, n ** 3).astype(np.float16).astype(np.float64)
    rhs[3::11] = -0.0
    rhs[::97] *= 1e-3
    stop = float(np.sqrt(np.sum(rhs * rhs)))
    spec = g.InnerSolverSpec(g.InnerMethod(method), 1e-9, 8, 5)

    def run():
        sysx = g.CudaGadiSystem(S)
        sysx.prepare(0.2, 1.0, g.Precision.Half, spec, g.Accum.Fp32)
        sysx.set_inner_stop_norm(stop)
        return sysx.solve_H(rhs) if method == CG else sysx.solve_S(rhs)

    x, it, st = run()
    monkeypatch.setenv("GADI_ST25H", "0")
    wx, wit, wst = run()
    monkeypatch.delenv("GADI_ST25H")
    assert (it, int(st)) == (wit, int(wst))
    assert same(x, wx)


def test_fast_path_whole_solve_n256_equals_generic(monkeypatch):
    """Three outer steps at n = 256 (C3's operator and inner mode): the fast
    binary16 passes, the speculative outer residual and the fused GMRES
    zero-start residual against the generic passes and the two-pass outer
    residual, bit for bit."""
    n = 256
    S = g.build_convdiff3d(n, r=0.0975)
    b = np.random.default_rng(3).uniform(-1, 1, n ** 3)
    cfg = g.GadiConfig(alpha=0.2, xi=1e-20, u_r=g.Precision.Half, accum=g.Accum.Fp32, max_outer_iters=3,
                       inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 5, 30))
    res = g.gadi_ir_solve(S, b, g.hss_split(S), cfg)
    monkeypatch.setenv("GADI_ST25H", "0")
    monkeypatch.setenv("GADI_NO_SPEC", "1")
    ref = g.gadi_ir_solve(S, b, g.hss_split(S), cfg)
    assert res.report.outer_iters == ref.report.outer_iters == 3
    assert res.report.inner_iter_totals == ref.report.inner_iter_totals
    assert same(res.x, ref.x)
    assert same(res.report.rel_residual_history, ref.report.rel_residual_history)


@pytest.mark.parametrize("n,fmt,accum", [(64, HALF, True), (64, SINGLE, False), (128, HALF, True)])
def test_resid64_variants_equal_st25(monkeypatch, n, fmt, accum):
    """The dedicated binary64 outer-residual kernel (k_resid64, n >= 64: both the
    two-pass PolResidA route of the first steps and the speculative PolResidSpec
    pass) against the generic k_st25 passes (GADI_R64=0, validated against the
    oracle at small n), for every compiled variant: x, history and counts bit for bit."""
    S = g.build_convdiff3d(n, r=0.0975)
    b = np.random.default_rng(5).uniform(-1, 1, n ** 3)
    b[7::13] *= 1e-6
    cfg = g.GadiConfig(alpha=0.3, xi=1e-20, u_r=g.Precision(fmt), max_outer_iters=6,
                       accum=g.Accum.Fp32 if accum else g.Accum.Native,
                       inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 5, 30))
    monkeypatch.setenv("GADI_R64", "0")
    ref = g.gadi_ir_solve(S, b, g.hss_split(S), cfg)
    for v in ("1", "2", "3", "4", "5"):
        monkeypatch.setenv("GADI_R64", v)
        res = g.gadi_ir_solve(S, b, g.hss_split(S), cfg)
        assert res.report.outer_iters == ref.report.outer_iters == 6
        assert same(res.x, ref.x), v
        assert same(res.report.rel_residual_history, ref.report.rel_residual_history), v
    monkeypatch.delenv("GADI_R64")


@pytest.mark.parametrize("eps,max_inner,restart", [(1e-9, 40, 12), (1e-12, 5, 30), (1e-6, 40, 5)])
def test_speculative_arnoldi_windows_equal_stepwise(monkeypatch, eps, max_inner, restart):
    """Fused-mode GMRES with the Arnoldi steps queued in windows of up to 8 (one
    host sync per window, 1/h formed on the device) against the step-by-step
    loop (GADI_GM_SPEC=0): windows that cross restarts, that end by convergence
    in mid-window, and the C3 shape (5 steps, one window) -- same x, counts, status."""
    n = 32
    S = g.build_convdiff3d(n, r=0.0975)
    rng = np.random.default_rng(17)
    rhs = rng.uniform(-1, 1, n ** 3).astype(np.float16).astype(np.float64)
    rhs[3::11] = -0.0
    stop = float(np.sqrt(np.sum(rhs * rhs)))
    spec = g.InnerSolverSpec(g.InnerMethod.Gmres, eps, max_inner, restart)

    def run():
        sysx = g.CudaGadiSystem(S)
        sysx.prepare(0.2, 1.0, g.Precision.Half, spec, g.Accum.Fp32)
        sysx.set_inner_stop_norm(stop)
        return sysx.solve_S(rhs)

    x, it, st = run()
    monkeypatch.setenv("GADI_GM_SPEC", "0")
    wx, wit, wst = run()
    monkeypatch.delenv("GADI_GM_SPEC")
    assert (it, int(st)) == (wit, int(wst))
    assert same(x, wx)


@pytest.mark.parametrize("kind,fmt,accum", [("stencil", HALF, True), ("stencil", SINGLE, False), ("stencil", DOUBLE, False),
                                            ("band", HALF, True)])
def test_cg_start_reuses_outer_sum_of_squares(orc, monkeypatch, kind, fmt, accum):
    """The H solve's start (k_cg_init) takes the binary64 ||rhat||^2 of its stop test from the
    outer pass that produced rhat (same values, same tree) and reduces only the inner-format
    dot. GADI_CHECK_SS makes the library reduce it again and throw if one bit differs, on
    stencil (n = 64: k_resid64; two-pass steps and speculative steps) and SELL systems; the
    solve must also equal the oracle's."""
    if kind == "stencil":
        n = 64 if fmt != DOUBLE else 16
        S, A = stencil_and_csr(orc, n, r=0.0975 if n == 64 else None)
        alpha = 0.3
    else:
        A = orc.band(8192, 26, 300, 4)
        S = g.build_band_csr(8192, 26, 300, 4)
        alpha = 3.0
    _, b = orc.make_rhs(A, 1, -1.0, 1.0)
    gcfg = g.GadiConfig(alpha=alpha, xi=1e-20, u_r=g.Precision(fmt), stall_window=400, max_outer_iters=8,
                        accum=g.Accum.Fp32 if accum else g.Accum.Native,
                        inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 5, 30))
    monkeypatch.setenv("GADI_CHECK_SS", "1")
    res = g.gadi_ir_solve(S, b, g.hss_split(S), gcfg)
    monkeypatch.delenv("GADI_CHECK_SS")
    cfg = Config.make(alpha=alpha, xi=1e-20, u_r=fmt, method=CG, tol_epsilon=1e-12, max_inner_iters=5,
                      stall_window=400, accum=1 if accum else 0, max_outer_iters=8)
    wx, wrep, _ = orc.solve(A, b, cfg)
    assert res.report.outer_iters == wrep.outer_iters
    assert same(res.x, wx)
