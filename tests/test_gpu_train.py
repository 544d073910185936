"""GPR training-set generation on the device (gadi_train.cu) against the
reference's alpha_bisection / generate_training_set (gpr.cpp:15-68): the
chosen alpha and its outer-iteration count are exactly the reference's
(golden vectors from the reference itself), because every probe is a
bitwise-reference solve and the choice follows the reference's probe order."""
import os

import numpy as np
import pytest

import paper_2501_04229_b200 as g

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


SETTINGS = {
    "bs6": dict(train_xi=1e-8, max_outer=1500),
    "bd5": dict(train_xi=1e-8, max_outer=800),
    "bh4": dict(train_xi=1e-3, max_outer=800),
    "bcg5": dict(max_outer=800, inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-6, 50, 30)),
}


@pytest.mark.parametrize("tag", list(SETTINGS))
def test_alpha_bisection_golden(gold, tag):
    n, fmt, lo, hi, budget, a, it = gold[f"bis_{tag}"]
    st = g.DichotomySettings(**SETTINGS[tag])
    alpha, iters = g.alpha_bisection(int(n), g.Precision(int(fmt)), lo, hi, int(budget), st)
    assert alpha == a and iters == int(it)


def test_generate_training_set_golden_and_deterministic(gold):
    """test_gpr.cpp:144-160: sizes {4,5,6}, single, budget 9; bitwise reproducible."""
    st = g.DichotomySettings(budget=9, train_xi=1e-8, max_outer=800)
    ts1 = g.generate_training_set([6, 4, 5], g.Precision.Single, st)
    ts2 = g.generate_training_set([4, 5, 6], g.Precision.Single, st)
    want = [gold[f"ts_{n}"] for n in (4, 5, 6)]
    for t in (ts1, ts2):
        assert [p.size_n for p in t.pairs] == [64, 125, 216]
        assert [p.alpha_opt for p in t.pairs] == [w[1] for w in want]
        assert [p.iters_at_opt for p in t.pairs] == [int(w[2]) for w in want]
    model = g.fit_training_set(ts1)
    ext = g.retrain_extend(model, ts1, [125, 512, 1000])
    assert [p.size_n for p in ext.pairs] == [64, 125, 216, 512, 1000]
    assert [p.iters_at_opt for p in ext.pairs][3:] == [0, 0]
    assert all(p.alpha_opt > 0 for p in ext.pairs)


def test_training_errors():
    st = g.DichotomySettings(train_xi=1e-8, max_outer=1500)
    with pytest.raises(g.ParameterError):
        g.alpha_bisection(6, g.Precision.Single, 5.0, 1.0, 7, st)
    with pytest.raises(g.ParameterError):
        g.alpha_bisection(6, g.Precision.Single, 0.1, 1.0, 2, st)
    # bracket squeezed into a non-convergent region (test_gpr.cpp:64-67)
    with pytest.raises(g.NoConvergentAlpha):
        g.alpha_bisection(6, g.Precision.Single, 1e-2, 2e-2, 3, g.DichotomySettings(train_xi=1e-8, max_outer=3))
    with pytest.raises(g.ParameterError):
        g.generate_training_set([4, 4], g.Precision.Single, g.DichotomySettings(budget=3, max_outer=800))
