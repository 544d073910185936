"""Sylvester GADI-AB on the device (gadi_sylv.cu) against the reference's own
gadi_ab_solve (sylvester.cpp:122-133) on build_sylvester (problems.cpp:45-66):
golden vectors from the reference (tests/golden/make_golden.py section 8).
Every pass restates the reference's arithmetic and order (u_f-rounded
residual fold, binary64 apply, sequential norm2_64, BandLU column/row solves),
so X, the residual history and the report are bit for bit the reference's."""
import os

import numpy as np
import pytest

import paper_2501_04229_b200 as g

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz")
P = g.Precision
CASES = {
    "s16": (16, 0.1, dict(alpha=0.5, xi=1e-22, max_outer_iters=20000)),
    "c7a": (64, 0.1, dict(alpha=0.02, xi=0.0, u_r=P.Half, max_outer_iters=30000, stall_window=400,
                          residual_scaling=False)),
    "c7b": (64, 1.0, dict(alpha=10.0, xi=0.0, u_r=P.Half, max_outer_iters=30000, stall_window=400,
                          residual_scaling=False)),
    "sgl": (24, 0.5, dict(alpha=0.3, xi=1e-12, u_r=P.Single, u=P.Single, u_f=P.Single, max_outer_iters=5000)),
}


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.mark.parametrize("tag", list(CASES))
def test_gadi_ab_solve_golden(gold, tag):
    n, r, kw = CASES[tag]
    res = g.gadi_ab_solve(g.build_sylvester(n, r), g.GadiConfig(**kw))
    rep = res.report
    assert [int(rep.status), rep.outer_iters, rep.inner_iter_totals, rep.inner_stagnations] == \
        list(gold[f"syl_{tag}_info"])
    X = res.X.T.reshape(-1)  # column-major vec
    assert np.array_equal(X.view(np.int64), gold[f"syl_{tag}_X"].view(np.int64))
    assert np.array_equal(rep.rel_residual_history.view(np.int64), gold[f"syl_{tag}_hist"].view(np.int64))


def test_identity_converges_immediately():
    """test_problems.cpp:139-150: A = B = I, C = -2: contraction 1/2, two steps to rres 1/4."""
    I6 = g.tridiag(6, 0.0, 1.0, 0.0)
    prob = g.SylvesterProblem(I6, I6, np.full((6, 6), -2.0), np.ones((6, 6)))
    res = g.gadi_ab_solve(prob, g.GadiConfig(alpha=1.0, xi=0.07))
    assert res.report.status == g.SolveStatus.Converged and res.report.outer_iters <= 2


def test_real_instance_solves():
    """test_problems.cpp:152-160: X = ones to 1e-7."""
    res = g.gadi_ab_solve(g.build_sylvester(16, 0.1), g.GadiConfig(alpha=0.5, xi=1e-22, max_outer_iters=20000))
    assert res.report.status == g.SolveStatus.Converged
    assert np.allclose(res.X, 1.0, rtol=1e-7, atol=0)
