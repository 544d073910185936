"""explicit_splitting (splitting.cpp:22-35) through the boundary.

tests/golden/explicit_split.npz holds the reference's gadi_ir_solve(A, b,
explicit_splitting(A, M, N), cfg) on build_convdiff3d(6) with three non-HSS
splittings (tests/golden/make_golden_split.py). CPU: the oracle restatement
(orc_solve_split: orc_explicit_check + orc_shift_diagonal) equals them bit for
bit. GPU: gadi_cuda_set_split(EXPLICIT, M, N) + gadi_cuda_solve equals them
bit for bit (histories to 1e-13: binary64 norm summation order), the M + N = A
check raises ContractViolation like the reference, and HSS can be restored.
"""
import importlib.util
import os

import numpy as np
import pytest

from oracle import CSR, Config

HERE = os.path.dirname(os.path.abspath(__file__))
_spec = importlib.util.spec_from_file_location("make_golden_split", os.path.join(HERE, "golden", "make_golden_split.py"))
mgs = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(mgs)
CASES = mgs.CASES


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(HERE, "golden", "explicit_split.npz"))


def same(a, b):
    return np.array_equal(np.ascontiguousarray(a, np.float64).view(np.int64),
                          np.ascontiguousarray(b, np.float64).view(np.int64))


def parts(gold, nm):
    n = len(gold["b"])
    return [CSR(n, gold[f"{nm}_{t}_rp"], gold[f"{nm}_{t}_ci"], gold[f"{nm}_{t}_v"]) for t in ("M", "N")]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_oracle_explicit_split_equals_reference(orc, gold, i):
    nm, ur, kw = CASES[i]
    A = orc.convdiff(6)
    M, N = parts(gold, nm)
    # the generator's splits are reproducible from the oracle alone
    M2, N2 = mgs.splits(orc, A)[nm]
    assert same(M.v, M2.v) and same(N.v, N2.v) and np.array_equal(N.ci, N2.ci)
    x, rep, hist = orc.solve(A, gold["b"], Config.make(u_r=ur, **kw), split=(M, N))
    assert [rep.status, rep.outer_iters, rep.inner_iter_totals, rep.inner_stagnations] == list(gold[f"case{i}_info"])
    assert same(x, gold[f"case{i}_x"])
    assert same(hist, gold[f"case{i}_hist"])


def test_oracle_explicit_check(orc, gold):
    A = orc.convdiff(6)
    M, N = parts(gold, "tri")
    bad = CSR(N.n, N.rp, N.ci, N.v.copy())
    bad.v[5] = np.nextafter(np.nextafter(bad.v[5], np.inf), np.inf)  # two ulps off
    with pytest.raises(ValueError):
        orc.solve(A, gold["b"], Config.make(alpha=0.5), split=(M, bad))


def test_live_reference_explicit_split(orc, ref, gold):
    A = orc.convdiff(6)
    M, N = parts(gold, "nodiag")
    cfg = Config.make(u_r=1, method=2, tol_epsilon=1e-6, max_inner_iters=25, restart=7, alpha=3.0, xi=1e-10,
                      max_outer_iters=300)
    xr, rr, hr = ref.solve_split(A, M, N, gold["b"], cfg)
    xo, ro, ho = orc.solve(A, gold["b"], cfg, split=(M, N))
    assert (rr.status, rr.outer_iters, rr.inner_iter_totals) == (ro.status, ro.outer_iters, ro.inner_iter_totals)
    assert same(xr, xo) and same(hr, ho)


# ------------------------------------------------------------------ device
@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(CASES)))
def test_device_explicit_split_equals_reference(orc, gold, i):
    import paper_2501_04229_b200 as g
    nm, ur, kw = CASES[i]
    A = orc.convdiff(6)
    Ag = g.SparseMatrix(A.n, A.n, A.rp, A.ci, A.v)
    M, N = [g.SparseMatrix(p.n, p.n, p.rp, p.ci, p.v) for p in parts(gold, nm)]
    kw = dict(kw)
    inner = g.InnerSolverSpec(g.InnerMethod(kw.pop("method")), kw.pop("tol_epsilon", 1e-2),
                              kw.pop("max_inner_iters", 1000), kw.pop("restart", 30))
    cfg = g.GadiConfig(u_r=g.Precision(ur), inner=inner, **kw)
    res = g.gadi_ir_solve(Ag, gold["b"], g.explicit_splitting(Ag, M, N), cfg)
    assert [int(res.report.status), res.report.outer_iters, res.report.inner_iter_totals,
            res.report.inner_stagnations] == list(gold[f"case{i}_info"])
    assert same(res.x, gold[f"case{i}_x"])
    np.testing.assert_allclose(res.report.rel_residual_history, gold[f"case{i}_hist"], rtol=1e-13, atol=0)


@pytest.mark.gpu
def test_device_explicit_split_contract_and_restore(orc, gold):
    import paper_2501_04229_b200 as g
    A = orc.convdiff(6)
    Ag = g.SparseMatrix(A.n, A.n, A.rp, A.ci, A.v)
    Mo, No = parts(gold, "tri")
    M = g.SparseMatrix(Mo.n, Mo.n, Mo.rp, Mo.ci, Mo.v)
    v = No.v.copy()
    v[5] = np.nextafter(np.nextafter(v[5], np.inf), np.inf)
    with pytest.raises(g.ContractViolation, match="M \\+ N != A"):
        g.gadi_ir_solve(Ag, gold["b"], g.explicit_splitting(Ag, M, g.SparseMatrix(No.n, No.n, No.rp, No.ci, v)),
                        g.GadiConfig(alpha=0.5))
    with pytest.raises(g.ContractViolation, match="shape mismatch"):
        g.explicit_splitting(Ag, M, g.SparseMatrix(3, 3, [0, 1, 2, 3], [0, 1, 2], [1.0, 1.0, 1.0]))
    st = g.build_convdiff3d(6)
    with pytest.raises(g.UnsupportedError):
        g.explicit_splitting(st, M, M)
    # one handle: explicit, then back to HSS -- the HSS solve equals a fresh handle's
    N = g.SparseMatrix(No.n, No.n, No.rp, No.ci, No.v)
    cfg = g.GadiConfig(alpha=0.5, xi=1e-12, u_r=g.Precision.Single)
    sysx = g.CudaGadiSystem(Ag, split=g.explicit_splitting(Ag, M, N))
    r1 = sysx.solve(gold["b"], cfg)
    assert same(r1.x, gold["case4_x"])
    sysx.set_split(g.hss_split(Ag))
    r2 = sysx.solve(gold["b"], cfg)
    sysx.close()
    r3 = g.gadi_ir_solve(Ag, gold["b"], g.hss_split(Ag), cfg)
    assert same(r2.x, r3.x) and r2.report.outer_iters == r3.report.outer_iters
    assert not same(r1.x, r2.x)
