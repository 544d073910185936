"""MatrixMarket ingest (matrix_market.cpp:22-86). CPU: the restatement
(oracle/mm.py) pinned to the reference's own reads of the fixtures
(tests/golden/mm_reference.npz, made by tests/golden/make_mm.py), and the
writer's text against the restatement. GPU: gadi_mm_read (host parse + device
from_triplets assembly) equals the reference bit for bit, errors included."""
import os

import numpy as np
import pytest

from oracle import mm

HERE = os.path.dirname(os.path.abspath(__file__))
MM = os.path.join(HERE, "golden", "mm")
FILES = sorted(f[:-4] for f in os.listdir(MM))


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(HERE, "golden", "mm_reference.npz"))


def check(gold, key, got):
    if isinstance(got, int):
        assert f"{key}_err" in gold.files and int(gold[f"{key}_err"][0]) == got, (key, got)
        return
    nr, nc, rp, ci, v = got
    assert [nr, nc] == list(gold[f"{key}_shape"])
    assert np.array_equal(rp, gold[f"{key}_rp"]) and np.array_equal(ci, gold[f"{key}_ci"])
    assert np.array_equal(np.asarray(v, np.float64).view(np.int64), gold[f"{key}_v"].view(np.int64))


@pytest.mark.parametrize("key", FILES)
def test_mm_restatement_pinned(gold, key):
    check(gold, key, mm.read(os.path.join(MM, key + ".mtx")))


@pytest.mark.parametrize("key", ["general", "symmetric", "skew", "integer", "empty"])
def test_mm_write_matches_restatement(tmp_path, key):
    """gadi_mm_write is host code (no device): its text is write_matrix_market's."""
    import paper_2501_04229_b200 as g
    nr, nc, rp, ci, v = mm.read(os.path.join(MM, key + ".mtx"))
    path = str(tmp_path / "out.mtx")
    g.write_matrix_market_file(path, g.SparseMatrix(nr, nc, rp, ci, v))
    assert open(path).read() == mm.write_text(nr, nc, rp, ci, v)
    back = mm.read(path)
    assert back[:2] == (nr, nc) and np.array_equal(back[2], rp) and np.array_equal(back[4], v)


@pytest.mark.gpu
@pytest.mark.parametrize("key", FILES)
def test_mm_read_device(gold, key):
    import paper_2501_04229_b200 as g
    try:
        A = g.read_matrix_market_file(os.path.join(MM, key + ".mtx"))
        got = (A.n_rows, A.n_cols, A.row_ptr, A.col_idx, A.values)
    except g.GadiError as e:
        got = type(e).code
    check(gold, key, got)


@pytest.mark.gpu
def test_mm_read_then_solve(orc, tmp_path):
    """A convdiff written to .mtx and read back solves exactly like the in-memory matrix."""
    import paper_2501_04229_b200 as g
    A = orc.convdiff(6)
    path = str(tmp_path / "cd6.mtx")
    g.write_matrix_market_file(path, g.SparseMatrix(A.n, A.n, A.rp, A.ci, A.v))
    B = g.read_matrix_market_file(path)
    assert np.array_equal(B.values.view(np.int64), A.v.view(np.int64)) and np.array_equal(B.col_idx, A.ci)
    _, b = orc.make_rhs(A, 0, 0.0, 1.0)
    cfg = g.GadiConfig(alpha=0.3, xi=1e-20, u_r=g.Precision.Single,
                       inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 50, 30))
    r1 = g.gadi_ir_solve(B, b, g.hss_split(B), cfg)
    A2 = g.SparseMatrix(A.n, A.n, A.rp, A.ci, A.v)
    r2 = g.gadi_ir_solve(A2, b, g.hss_split(A2), cfg)
    assert r1.report.outer_iters == r2.report.outer_iters and np.array_equal(r1.x, r2.x)
