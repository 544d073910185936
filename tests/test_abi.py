"""The C ABI boundary (include/gadi_cuda.h) without a GPU: the library loads,
exports every declared entry point, and the host-side contract (defaults,
validation, error codes) matches the reference's (solver.hpp:17-38,
solver.cpp:12-40, inner_solver.hpp:20-25)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2501_04229_b200 as g

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "gadi_cuda.h")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*[A-Za-z_][\w\s\*]*?\b(gadi_\w+)\s*\(", src, flags=re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    L = g.lib()
    names = declared()
    assert len(names) >= 25, names
    out = subprocess.run(["nm", "-D", "--defined-only", g.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (gadi_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert getattr(L, n) is not None


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", g.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_defaults_match_reference():
    L = g.lib()
    c = g._Config()
    L.gadi_config_default(C.byref(c))
    ref = g.GadiConfig()  # mirrors solver.hpp:17-38 / inner_solver.hpp:20-25
    assert (c.alpha, c.omega, c.xi) == (1.0, 1.0, 0.0) == (ref.alpha, ref.omega, ref.xi)
    assert (c.u_r, c.u, c.u_f) == (2, 2, 2)
    assert (c.inner.method, c.inner.tol_epsilon, c.inner.max_inner_iters, c.inner.restart) == (0, 1e-2, 1000, 30)
    assert (c.max_outer_iters, c.divergence_factor, c.stall_window) == (20000, 1e6, 0)
    assert (c.ones_start, c.residual_scaling) == (0, 1)
    assert ref.inner.method == g.InnerMethod.LuDirect and ref.max_outer_iters == 20000


def test_default_xi_and_status_names():
    L = g.lib()
    assert [L.gadi_default_xi(p) for p in (2, 1, 0)] == [1e-26, 1e-8, 1e-4]  # solver.cpp:12-18
    names = [L.gadi_status_name(s).decode() for s in range(6)]
    assert names == ["Converged", "MaxIters", "Diverged", "OverflowDetected", "SingularInPrecision", "Stalled"]
    assert L.gadi_abi_version() == 1


def test_enums_match_reference_numbering():
    assert [int(p) for p in g.Precision] == [0, 1, 2]          # precision.hpp:14
    assert [int(m) for m in g.InnerMethod] == [0, 1, 2]        # inner_solver.hpp:15
    assert [s.name for s in g.SolveStatus] == ["Converged", "MaxIters", "Diverged", "OverflowDetected",
                                               "SingularInPrecision", "Stalled"]  # solver.hpp:44-51
    assert [s.name for s in g.InnerStatus] == ["Converged", "Stagnated", "Overflow"]


def test_contract_errors_without_device():
    """Null arguments are contract violations, reported before any device work."""
    L = g.lib()
    assert L.gadi_cuda_create(None, None, None) == -1
    assert L.gadi_cuda_dim(None, None) == -1
    assert L.gadi_cuda_history(None, None, 0) == -1
    assert L.gadi_cuda_set_inner_stop_norm(None, 1.0) == -1
    assert L.gadi_cuda_destroy(None) == 0


def test_python_mirror_raises_reference_exceptions():
    A = g.build_convdiff3d(4)
    with pytest.raises(g.ContractViolation):
        g.gadi_ir_solve(A, [0.0] * 3, g.hss_split(A), g.GadiConfig())  # solver.cpp:252-253
    B = g.build_convdiff3d(4)
    with pytest.raises(g.ContractViolation):
        g.gadi_ir_solve(A, [0.0] * 64, g.hss_split(B), g.GadiConfig())
    assert issubclass(g.ParameterError, g.ContractViolation)  # errors.hpp:14-16


def test_build_convdiff3d_coefficients():
    S = g.build_convdiff3d(32)  # problems.hpp:16-22, r = 1/(2n+2)
    r = 1.0 / 66.0
    assert (S.t1, S.t2, S.t3) == (6.0, -1.0 - r, -1.0 + r)
    S2 = g.build_convdiff3d(512, beta=100.0)  # BASELINE configs[2]: r = beta h / 2
    assert S2.t2 == -1.0 - 100.0 / 1026.0


def test_training_csv_round_trip():
    """write_training_csv / read_training_csv (gpr.cpp:188-218): %.17g alphas survive."""
    import io
    import paper_2501_04229_b200 as g
    ts = g.TrainingSet([g.TrainingPair(64, 0.1 + 1e-17 * 3, 12), g.TrainingPair(125, 1 / 3, 0)],
                       g.Precision.Double)
    buf = io.StringIO()
    g.write_training_csv(buf, ts)
    assert buf.getvalue().splitlines()[0] == "n,alpha,iters,precision"
    back = g.read_training_csv(io.StringIO(buf.getvalue()))
    assert back == ts


def test_build_sylvester_mirror():
    """build_sylvester (problems.cpp:45-66): tridiagonal A = B, C = -(row + column sums)."""
    import paper_2501_04229_b200 as g
    p = g.build_sylvester(5, 0.5)
    sh = 100.0 / 36.0
    assert p.A.nnz() == 13 and p.A.values[0] == 2.0 + sh and p.A.values[1] == -1.0 + 0.5
    dense = np.zeros((5, 5))
    for i in range(5):
        for k in range(p.A.row_ptr[i], p.A.row_ptr[i + 1]):
            dense[i, p.A.col_idx[k]] = p.A.values[k]
    assert np.allclose(dense @ np.ones((5, 5)) + np.ones((5, 5)) @ dense + p.C_rhs, 0.0, atol=1e-13)
