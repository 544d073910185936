"""B200-native GADI-IR solver (sm_100a) — Python mirror of the reference API.

The compute path is ``libgadi_cuda.so`` (hand-written CUDA for sm_100a, built
in-tree from ``csrc/``) behind the C ABI in ``include/gadi_cuda.h``. This
module is a thin ctypes layer that mirrors the reference's C++ surface
(/root/reference/proj/core/include/gadi/solver.hpp, inner_solver.hpp,
problems.hpp, gpr.hpp) so that callers and tests read like the reference's:

    reference (C++)                         here (Python)
    GadiConfig / InnerSolverSpec            GadiConfig / InnerSolverSpec
    SolveStatus / SolveReport / GadiResult  SolveStatus / SolveReport / GadiResult
    build_convdiff3d({n})                   build_convdiff3d(n, r=None)  (matrix free)
    hss_split(A)                            hss_split(A)
    gadi_ir_solve(A, b, split, cfg, x0)     gadi_ir_solve(A, b, split, cfg, x0)
    class GadiSystem (6 virtuals)           CudaGadiSystem
    fit / predict_alpha                     gpr_fit / GprModel.predict

There is no CPU fallback: every entry point raises if the library or a CUDA
device is missing.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgadi_cuda.so")

__all__ = [
    "Precision", "InnerMethod", "SolveStatus", "InnerStatus", "Accum", "InnerSolverSpec", "GadiConfig",
    "SolveReport", "GadiResult", "SparseMatrix", "Stencil7", "Splitting", "build_convdiff3d",
    "hss_split", "gadi_ir_solve", "CudaGadiSystem", "GadiError", "ContractViolation", "ParameterError",
    "UnsupportedError", "FitError", "default_xi", "lib", "gpr_fit", "ShardGroup", "ShardSystem", "solve_group",
    "nccl_unique_id",
]


class Precision(enum.IntEnum):  # precision.hpp:14
    Half = 0
    Single = 1
    Double = 2


class InnerMethod(enum.IntEnum):  # inner_solver.hpp:15
    LuDirect = 0
    Cg = 1
    Gmres = 2


class SolveStatus(enum.IntEnum):  # solver.hpp:44-51
    Converged = 0
    MaxIters = 1
    Diverged = 2
    OverflowDetected = 3
    SingularInPrecision = 4
    Stalled = 5


class InnerStatus(enum.IntEnum):  # inner_solver.hpp:45
    Converged = 0
    Stagnated = 1
    Overflow = 2


class Accum(enum.IntEnum):
    Native = 0  # every op rounded to u_r (the reference's semantics)
    Fp32 = 1    # u_r storage, binary32 arithmetic and accumulation


# ---------------------------------------------------------------- errors
class GadiError(RuntimeError):
    code = -5


class ContractViolation(GadiError, ValueError):  # errors.hpp:9-12
    code = -1


class ParameterError(ContractViolation):  # errors.hpp:14-16
    code = -2


class UnsupportedError(GadiError):
    code = -3


class FitError(GadiError):  # errors.hpp:40-42
    code = -4


class SingularInPrecision(GadiError):  # errors.hpp: thrown by prepare (band_lu.cpp:106-108)
    code = -9


class OverflowDetected(GadiError):  # errors.hpp: thrown by prepare (band_lu.cpp:132-134)
    code = -10


class NoConvergentAlpha(GadiError):  # errors.hpp:35-37, alpha_bisection (gpr.cpp:45-48)
    code = -11


class IoError(GadiError):  # errors.hpp:43-45 (MatrixMarket files)
    code = -12


_ERRS = {-1: ContractViolation, -2: ParameterError, -3: UnsupportedError, -4: FitError,
         -9: SingularInPrecision, -10: OverflowDetected, -11: NoConvergentAlpha, -12: IoError}


# ---------------------------------------------------------------- ctypes structs
class _InnerSpec(C.Structure):
    _fields_ = [("method", C.c_int32), ("tol_epsilon", C.c_double),
                ("max_inner_iters", C.c_int32), ("restart", C.c_int32)]


class _Config(C.Structure):
    _fields_ = [("alpha", C.c_double), ("omega", C.c_double), ("xi", C.c_double),
                ("u_r", C.c_int32), ("u", C.c_int32), ("u_f", C.c_int32), ("inner", _InnerSpec),
                ("max_outer_iters", C.c_int32), ("divergence_factor", C.c_double),
                ("stall_window", C.c_int32), ("ones_start", C.c_int32),
                ("residual_scaling", C.c_int32), ("accum", C.c_int32)]


class _Report(C.Structure):
    _fields_ = [("status", C.c_int32), ("outer_iters", C.c_int32), ("final_rres", C.c_double),
                ("inner_iter_totals", C.c_int64), ("inner_stagnations", C.c_int32),
                ("history_len", C.c_int32), ("h_iters", C.c_int64), ("s_iters", C.c_int64),
                ("solve_ms", C.c_double), ("h_ms", C.c_double), ("s_ms", C.c_double),
                ("outer_ms", C.c_double), ("h2d_bytes", C.c_double), ("d2h_bytes", C.c_double),
                ("e2e_ms", C.c_double), ("launches", C.c_int64)]


class _Problem(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int64), ("t1", C.c_double), ("t2", C.c_double),
                ("t3", C.c_double), ("n_rows", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.POINTER(C.c_int64)), ("col_idx", C.POINTER(C.c_int64)),
                ("values", C.POINTER(C.c_double)), ("band", C.c_int64), ("k_off", C.c_int32),
                ("seed", C.c_uint64)]


class _CsrDesc(C.Structure):  # gadi_csr_desc
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.POINTER(C.c_int64)), ("col_idx", C.POINTER(C.c_int64)),
                ("values", C.POINTER(C.c_double))]


class _DevOpts(C.Structure):
    _fields_ = [("device", C.c_int32)]


class _Dichotomy(C.Structure):
    _fields_ = [("alpha_lo", C.c_double), ("alpha_hi", C.c_double), ("budget", C.c_int32),
                ("train_xi", C.c_double), ("max_outer", C.c_int32), ("inner", _InnerSpec)]


class _GprOpts(C.Structure):
    _fields_ = [("fixed_hypers", C.c_int32), ("sigma_f2", C.c_double), ("length", C.c_double),
                ("sigma_n2", C.c_double), ("has_sigma_n2", C.c_int32), ("device", C.c_int32)]


_f64p = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_lib = None


def lib():
    """Load libgadi_cuda.so (built in-tree). Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                          f"(make -C {os.path.join(HERE, 'csrc')}); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    L.gadi_config_default.argtypes = [C.POINTER(_Config)]
    L.gadi_config_default.restype = None
    L.gadi_default_xi.restype = C.c_double
    L.gadi_default_xi.argtypes = [C.c_int32]
    L.gadi_status_name.restype = C.c_char_p
    L.gadi_last_error.restype = C.c_char_p
    L.gadi_abi_version.restype = C.c_int32
    L.gadi_cuda_create.argtypes = [C.POINTER(_Problem), C.POINTER(_DevOpts), C.POINTER(C.c_void_p)]
    L.gadi_cuda_destroy.argtypes = [C.c_void_p]
    L.gadi_cuda_dim.argtypes = [C.c_void_p, _i64p]
    L.gadi_cuda_set_split.argtypes = [C.c_void_p, C.c_int32, C.POINTER(_CsrDesc), C.POINTER(_CsrDesc)]
    L.gadi_cuda_set_rhs.argtypes = [C.c_void_p, _f64p]
    L.gadi_cuda_residual_uf.argtypes = [C.c_void_p, C.c_int32, _f64p, _f64p]
    L.gadi_cuda_true_residual_norm.argtypes = [C.c_void_p, _f64p, _f64p]
    L.gadi_cuda_prepare.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int32, C.POINTER(_InnerSpec),
                                    C.c_int32]
    L.gadi_cuda_set_inner_stop_norm.argtypes = [C.c_void_p, C.c_double]
    L.gadi_cuda_reset.argtypes = [C.c_void_p]
    for f in ("gadi_cuda_solve_H", "gadi_cuda_solve_S"):
        getattr(L, f).argtypes = [C.c_void_p, _f64p, _f64p, _i32p, _i32p]
    L.gadi_cuda_solve.argtypes = [C.c_void_p, C.POINTER(_Config), _f64p, _f64p, _f64p, C.POINTER(_Report)]
    L.gadi_cuda_solve_device.argtypes = [C.c_void_p, C.POINTER(_Config), C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.POINTER(_Report)]
    L.gadi_cuda_history.argtypes = [C.c_void_p, _f64p, C.c_int32]
    L.gadi_cuda_apply.argtypes = [C.c_void_p, C.c_int32, _f64p, _f64p]
    L.gadi_cuda_dot.argtypes = [C.c_int32, C.c_int32, _f64p, _f64p, C.c_int64, _f64p]
    L.gadi_cuda_norm2.argtypes = [C.c_int32, C.c_int32, _f64p, C.c_int64, _f64p]
    L.gadi_cuda_make_rhs.argtypes = [C.c_void_p, C.c_uint64, C.c_double, C.c_double, C.c_void_p, C.c_void_p]
    L.gadi_gpr_fit.argtypes = [_f64p, _f64p, C.c_int32, C.POINTER(_GprOpts), C.POINTER(C.c_void_p)]
    L.gadi_gpr_predict.argtypes = [C.c_void_p, _f64p, C.c_int32, _f64p, _f64p]
    L.gadi_gpr_params.argtypes = [C.c_void_p, _f64p, _f64p, _f64p, _f64p, _f64p]
    L.gadi_gpr_destroy.argtypes = [C.c_void_p]
    L.gadi_gpr_timings.argtypes = [C.c_void_p, _f64p, _f64p, _f64p, _i32p, _i64p]
    L.gadi_cuda_launch_count.argtypes = [C.c_void_p]
    L.gadi_cuda_launch_count.restype = C.c_int64
    L.gadi_cuda_nnz.argtypes = [C.c_void_p, _i64p, _i64p]
    L.gadi_group_local.argtypes = [C.c_int32, C.POINTER(C.c_void_p)]
    L.gadi_nccl_unique_id.argtypes = [C.c_char_p]
    L.gadi_group_nccl.argtypes = [C.c_int32, C.c_int32, C.c_char_p, C.POINTER(C.c_void_p)]
    L.gadi_group_ipc.argtypes = [C.c_int32, C.c_int32, C.c_char_p, C.POINTER(C.c_void_p)]
    L.gadi_group_destroy.argtypes = [C.c_void_p]
    L.gadi_cuda_create_shard.argtypes = [C.POINTER(_Problem), C.POINTER(_DevOpts), C.c_void_p, C.c_int32,
                                         C.POINTER(C.c_void_p)]
    L.gadi_cuda_shard_range.argtypes = [C.c_void_p, _i64p, _i64p]
    L.gadi_cuda_solve_group.argtypes = [C.POINTER(C.c_void_p), C.c_int32, C.POINTER(_Config),
                                        C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                        C.POINTER(_Report)]
    L.gadi_dichotomy_default.argtypes = [C.POINTER(_Dichotomy)]
    L.gadi_dichotomy_default.restype = None
    L.gadi_alpha_bisection.argtypes = [C.c_int64, C.c_int32, C.c_double, C.c_double, C.c_int32,
                                       C.POINTER(_Dichotomy), C.c_int32, _f64p, _i32p]
    L.gadi_generate_training_set.argtypes = [_i64p, C.c_int32, C.c_int32, C.POINTER(_Dichotomy), C.c_int32,
                                             _i64p, _f64p, _i32p]
    L.gadi_mm_read.argtypes = [C.c_char_p, C.c_int32, C.POINTER(C.c_void_p)]
    L.gadi_csr_view.argtypes = [C.c_void_p, _i64p, _i64p, _i64p, C.POINTER(_i64p), C.POINTER(_i64p),
                                C.POINTER(_f64p)]
    L.gadi_csr_destroy.argtypes = [C.c_void_p]
    L.gadi_mm_write.argtypes = [C.c_char_p, C.c_int64, C.c_int64, _i64p, _i64p, _f64p]
    L.gadi_sylv_create.argtypes = [C.c_int64, _i64p, _i64p, _f64p, C.c_int64, _i64p, _i64p, _f64p, _f64p,
                                   C.c_int32, C.POINTER(C.c_void_p)]
    L.gadi_sylv_solve.argtypes = [C.c_void_p, C.POINTER(_Config), _f64p, _f64p, C.POINTER(_Report)]
    L.gadi_sylv_history.argtypes = [C.c_void_p, _f64p, C.c_int32]
    L.gadi_sylv_destroy.argtypes = [C.c_void_p]
    _lib = L
    return L


def _check(rc):
    if rc < 0:
        msg = lib().gadi_last_error().decode(errors="replace")
        raise _ERRS.get(rc, GadiError)(f"gadi error {rc}: {msg}")
    return rc


def _p(a, t=_f64p):
    return None if a is None else a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------- config / report
@dataclass
class InnerSolverSpec:  # inner_solver.hpp:20-25
    method: InnerMethod = InnerMethod.LuDirect
    tol_epsilon: float = 1e-2
    max_inner_iters: int = 1000
    restart: int = 30

    def _c(self):
        return _InnerSpec(int(self.method), self.tol_epsilon, self.max_inner_iters, self.restart)


@dataclass
class GadiConfig:  # solver.hpp:17-38
    alpha: float = 1.0
    omega: float = 1.0
    xi: float = 0.0
    u_r: Precision = Precision.Double
    u: Precision = Precision.Double
    u_f: Precision = Precision.Double
    inner: InnerSolverSpec = field(default_factory=InnerSolverSpec)
    max_outer_iters: int = 20000
    divergence_factor: float = 1e6
    stall_window: int = 0
    ones_start: bool = False
    residual_scaling: bool = True
    accum: Accum = Accum.Native  # extension (include/gadi_cuda.h)

    def _c(self):
        return _Config(self.alpha, self.omega, self.xi, int(self.u_r), int(self.u), int(self.u_f),
                       self.inner._c(), self.max_outer_iters, self.divergence_factor, self.stall_window,
                       int(self.ones_start), int(self.residual_scaling), int(self.accum))


def default_xi(u: Precision) -> float:  # solver.cpp:12-18
    return lib().gadi_default_xi(int(u))


@dataclass
class SolveReport:  # solver.hpp:54-64
    status: SolveStatus = SolveStatus.MaxIters
    outer_iters: int = 0
    rel_residual_history: np.ndarray = field(default_factory=lambda: np.ones(1))
    final_rres: float = 1.0
    inner_iter_totals: int = 0
    inner_stagnations: int = 0
    h_iters: int = 0
    s_iters: int = 0
    solve_ms: float = 0.0
    h_ms: float = 0.0
    s_ms: float = 0.0
    h2d_bytes: float = 0.0
    d2h_bytes: float = 0.0
    outer_ms: float = 0.0
    e2e_ms: float = 0.0
    launches: int = 0


@dataclass
class GadiResult:  # solver.hpp:66-69
    x: np.ndarray
    report: SolveReport


# ---------------------------------------------------------------- problems
class SparseMatrix:
    """CSR with the reference's layout (sparse.hpp:17-65): int64 row_ptr /
    col_idx (strictly increasing per row), binary64 values."""

    def __init__(self, n_rows, n_cols, row_ptr, col_idx, values):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, np.int64)
        self.values = _f64(values)

    def nnz(self):
        return int(self.row_ptr[-1])

    def _desc(self):
        return _Problem(1, 0, 0.0, 0.0, 0.0, self.n_rows, self.nnz(), _p(self.row_ptr, _i64p),
                        _p(self.col_idx, _i64p), _p(self.values))


@dataclass
class Stencil7:
    """The 3D convection-diffusion operator of build_convdiff3d
    (problems.cpp:8-43), matrix free: n per direction, coefficients t1 (diag),
    t2 (i-1, j-1, k-1), t3 (k+1, j+1, i+1)."""
    n: int
    t1: float
    t2: float
    t3: float

    @property
    def n_rows(self):
        return self.n ** 3

    def _desc(self):
        return _Problem(0, self.n, self.t1, self.t2, self.t3, 0, 0, None, None, None)


@dataclass
class BandRandom:
    """BASELINE configs[3], generated on the device: n_rows rows with k_off
    distinct off-diagonal columns uniform within +-band of the diagonal,
    values U[-1,1], diagonal 1.1 * row abs sum (strictly diagonally dominant,
    H positive definite); splitmix64 stream `seed` (oracle: orc_band_csr)."""
    n_rows: int
    k_off: int = 26
    band: int = 4096
    seed: int = 2

    def _desc(self):
        return _Problem(2, 0, 0.0, 0.0, 0.0, self.n_rows, 0, None, None, None, self.band, self.k_off, self.seed)


def build_band_csr(n_rows: int, k_off: int = 26, band: int = 4096, seed: int = 2) -> BandRandom:
    return BandRandom(n_rows, k_off, band, seed)


def build_convdiff3d(n: int, r: Optional[float] = None, beta: Optional[float] = None) -> Stencil7:
    """problems.hpp:16-22: t1 = 6, t2 = -1 - r, t3 = -1 + r with r = 1/(2n+2)
    (beta = 1). beta (BASELINE configs) gives r = beta * h / 2, h = 1/(n+1)."""
    if r is None:
        r = (1.0 if beta is None else beta) / (2.0 * n + 2.0)
    return Stencil7(n, 6.0, -1.0 - r, -1.0 + r)


@dataclass
class Splitting:  # splitting.hpp:17-22; the HSS split is built on the device
    A: object
    kind: str = "hss"            # SplitKind: "hss" | "explicit"
    M: Optional["SparseMatrix"] = None
    N: Optional["SparseMatrix"] = None


def hss_split(A) -> Splitting:
    """M = (A+A^T)/2, N = (A-A^T)/2 (splitting.cpp:12-20); the device builds it."""
    return Splitting(A, "hss")


def explicit_splitting(A, M: "SparseMatrix", N: "SparseMatrix") -> Splitting:
    """User-supplied splitting A = M + N (splitting.cpp:22-35). Shapes are
    checked here; the one-ulp M + N = A check runs in gadi_cuda_set_split when
    the split is bound to a handle (ContractViolation "M + N != A")."""
    if not isinstance(A, SparseMatrix):
        raise UnsupportedError("explicit_splitting: A must be a SparseMatrix (CSR)")
    if (M.n_rows != A.n_rows or N.n_rows != A.n_rows or M.n_cols != A.n_cols or N.n_cols != A.n_cols):
        raise ContractViolation("explicit_splitting: shape mismatch")
    return Splitting(A, "explicit", M, N)


# ---------------------------------------------------------------- GadiSystem mirror
class CudaGadiSystem:
    """The reference's GadiSystem plugin (solver.hpp:74-89) on the device.

    Holds one handle: the operator A in device memory, its HSS split, and the
    inner engines built by prepare(). Vectors cross the boundary as binary64
    numpy arrays like the reference's Vector.
    """

    def __init__(self, A, b=None, device: int = 0, split: Optional[Splitting] = None):
        L = lib()
        self._h = C.c_void_p()
        self._A = A
        desc = A._desc()
        _check(L.gadi_cuda_create(C.byref(desc), C.byref(_DevOpts(device)), C.byref(self._h)))
        n = C.c_int64()
        L.gadi_cuda_dim(self._h, C.byref(n))
        self.n = n.value
        if split is not None:
            try:
                self.set_split(split)
            except Exception:
                self.close()
                raise
        if b is not None:
            self.set_rhs(b)

    def set_split(self, split: Splitting):
        """Bind the splitting the solves use (the `split` argument of
        gadi_ir_solve, solver.hpp:97-98): hss_split(A) or explicit_splitting(A, M, N)."""
        if split.A is not self._A:
            raise ContractViolation("set_split: split does not belong to A")
        if split.kind == "hss":
            _check(lib().gadi_cuda_set_split(self._h, 0, None, None))
            return
        d = []
        for m in (split.M, split.N):
            d.append(_CsrDesc(m.n_rows, m.n_cols, m.nnz(), _p(m.row_ptr, _i64p), _p(m.col_idx, _i64p), _p(m.values)))
        _check(lib().gadi_cuda_set_split(self._h, 1, C.byref(d[0]), C.byref(d[1])))

    def close(self):
        if self._h:
            lib().gadi_cuda_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def dim(self):
        return self.n

    def nnz(self):
        """(stored entries of A, of the H/S union pattern); (0, 0) for stencils."""
        a, hs = C.c_int64(), C.c_int64()
        _check(lib().gadi_cuda_nnz(self._h, C.byref(a), C.byref(hs)))
        return a.value, hs.value

    def set_rhs(self, b):
        self._b = _f64(b)
        _check(lib().gadi_cuda_set_rhs(self._h, _p(self._b)))

    def residual_uf(self, x, u_f: Precision = Precision.Double):
        x = _f64(x)
        s = np.empty(self.n)
        _check(lib().gadi_cuda_residual_uf(self._h, int(u_f), _p(x), _p(s)))
        return s

    def true_residual_norm(self, x) -> float:
        x = _f64(x)
        out = C.c_double()
        _check(lib().gadi_cuda_true_residual_norm(self._h, _p(x), C.byref(out)))
        return out.value

    def prepare(self, alpha, omega, u_r: Precision, spec: InnerSolverSpec, accum: Accum = Accum.Native):
        _check(lib().gadi_cuda_prepare(self._h, alpha, omega, int(u_r), C.byref(spec._c()), int(accum)))

    def reset(self):
        """Drop the prepared inner state: the next solve re-runs prepare (factorizations included)."""
        _check(lib().gadi_cuda_reset(self._h))

    def set_inner_stop_norm(self, s):
        _check(lib().gadi_cuda_set_inner_stop_norm(self._h, s))

    def _inner(self, f, rhs):
        rhs = _f64(rhs)
        x = np.empty(self.n)
        it, st = C.c_int32(), C.c_int32()
        _check(f(self._h, _p(rhs), _p(x), C.byref(it), C.byref(st)))
        return x, it.value, InnerStatus(st.value)

    def solve_H(self, rhat):
        return self._inner(lib().gadi_cuda_solve_H, rhat)

    def solve_S(self, pz):
        return self._inner(lib().gadi_cuda_solve_S, pz)

    def apply(self, which: str, x):
        """y = A x (binary64 fold), H x or S x (inner arithmetic, after prepare)."""
        x = _f64(x)
        y = np.empty(self.n)
        _check(lib().gadi_cuda_apply(self._h, {"A": 0, "H": 1, "S": 2}[which], _p(x), _p(y)))
        return y

    def solve(self, b, cfg: GadiConfig, x0=None) -> GadiResult:
        """gadi_ir_solve's body (solver.hpp:97-98): host b/x0 in, host x out."""
        b = _f64(b)
        x0a = None if x0 is None else _f64(x0)
        x = np.empty(self.n)
        rep = _Report()
        _check(lib().gadi_cuda_solve(self._h, C.byref(cfg._c()), _p(b), _p(x0a), _p(x), C.byref(rep)))
        return GadiResult(x, self._report(rep))

    def solve_into(self, b: np.ndarray, x_out: np.ndarray, cfg: GadiConfig, x0=None) -> SolveReport:
        """solve() into a caller buffer (e.g. pinned host memory); b, x_out
        must be contiguous float64 arrays of length dim()."""
        if b.dtype != np.float64 or x_out.dtype != np.float64 or len(b) != self.n or len(x_out) != self.n:
            raise ContractViolation("solve_into: b and x_out must be float64 of length dim()")
        x0a = None if x0 is None else _f64(x0)
        rep = _Report()
        _check(lib().gadi_cuda_solve(self._h, C.byref(cfg._c()), _p(b), _p(x0a), _p(x_out), C.byref(rep)))
        return self._report(rep)

    def solve_device(self, d_b: int, d_x: int, cfg: GadiConfig, d_x0: int = 0) -> SolveReport:
        """Same loop on device pointers (e.g. torch tensors' data_ptr())."""
        rep = _Report()
        _check(lib().gadi_cuda_solve_device(self._h, C.byref(cfg._c()), C.c_void_p(d_b),
                                            C.c_void_p(d_x0 or None), C.c_void_p(d_x), C.byref(rep)))
        return self._report(rep)

    def make_rhs(self, seed: int, lo: float, hi: float, d_xtrue: int, d_b: int):
        _check(lib().gadi_cuda_make_rhs(self._h, seed, lo, hi, C.c_void_p(d_xtrue), C.c_void_p(d_b)))

    def _report(self, rep: _Report) -> SolveReport:
        hist = np.empty(max(rep.history_len, 1))
        got = lib().gadi_cuda_history(self._h, _p(hist), len(hist))
        return SolveReport(SolveStatus(rep.status), rep.outer_iters, hist[:got].copy(), rep.final_rres,
                           rep.inner_iter_totals, rep.inner_stagnations, rep.h_iters, rep.s_iters,
                           rep.solve_ms, rep.h_ms, rep.s_ms, rep.h2d_bytes, rep.d2h_bytes, rep.outer_ms,
                           rep.e2e_ms, rep.launches)


class ShardGroup:
    """A sharded (z-slab) solve's communicator, SURVEY §8(e) (include/gadi_cuda.h).

    ShardGroup.local(world): the ranks are threads of this process (one or
    several devices; solve them together with solve_group).
    ShardGroup.nccl(world, rank, uid): one rank per process over NCCL; every
    process passes the same 128-byte id (nccl_unique_id() on one rank,
    broadcast by the caller) and solves its shard collectively.
    """

    def __init__(self, ptr, world):
        self._g, self.world = ptr, world

    @classmethod
    def local(cls, world: int) -> "ShardGroup":
        g = C.c_void_p()
        _check(lib().gadi_group_local(world, C.byref(g)))
        return cls(g, world)

    @classmethod
    def nccl(cls, world: int, rank: int, uid: bytes) -> "ShardGroup":
        if len(uid) != 128:
            raise ContractViolation("nccl id must be 128 bytes")
        g = C.c_void_p()
        _check(lib().gadi_group_nccl(world, rank, uid, C.byref(g)))
        return cls(g, world)

    @classmethod
    def ipc(cls, world: int, rank: int, name: str) -> "ShardGroup":
        """One rank per process on one node over CUDA IPC (gadi_group_ipc): `name`
        is a POSIX shared-memory name ("/..."), the same on every rank. Collective."""
        g = C.c_void_p()
        _check(lib().gadi_group_ipc(world, rank, name.encode(), C.byref(g)))
        return cls(g, world)

    def close(self):
        if self._g:
            lib().gadi_group_destroy(self._g)
            self._g = C.c_void_p()


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().gadi_nccl_unique_id(buf))
    return buf.raw


class ShardSystem(CudaGadiSystem):
    """One rank's z-slab of a 7-point stencil problem (gadi_cuda_create_shard).
    Vectors are the shard's rows [first_row, first_row + n)."""

    def __init__(self, A: "Stencil7", group: ShardGroup, rank: int, device: int = 0):
        L = lib()
        self._h = C.c_void_p()
        self._A, self.group, self.rank = A, group, rank
        desc = A._desc()
        _check(L.gadi_cuda_create_shard(C.byref(desc), C.byref(_DevOpts(device)), group._g, rank,
                                        C.byref(self._h)))
        first, n = C.c_int64(), C.c_int64()
        _check(L.gadi_cuda_shard_range(self._h, C.byref(first), C.byref(n)))
        self.first_row, self.n = first.value, n.value


def solve_group(shards, cfg: GadiConfig, d_b, d_x, d_x0=None):
    """A local group's sharded solve (gadi_cuda_solve_group): shards[r] is
    rank r; d_b / d_x / d_x0 are per-rank device pointers. One report per rank."""
    w = len(shards)
    hs = (C.c_void_p * w)(*[s_._h for s_ in shards])
    arr = lambda ptrs: (C.c_void_p * w)(*[C.c_void_p(p) for p in ptrs])
    reps = (_Report * w)()
    _check(lib().gadi_cuda_solve_group(hs, w, C.byref(cfg._c()), arr(d_b), None if d_x0 is None else arr(d_x0),
                                       arr(d_x), reps))
    return [sh._report(reps[r]) for r, sh in enumerate(shards)]


def gadi_ir_solve(A, b, split: Splitting, cfg: GadiConfig, x0=None, device: int = 0) -> GadiResult:
    """gadi_ir_solve (solver.hpp:97-98; solver.cpp:250-258) on the device."""
    if split.A is not A:
        raise ContractViolation("gadi_ir_solve: split does not belong to A")
    if len(b) != A.n_rows:
        raise ContractViolation("gadi_ir_solve: dimension mismatch")  # solver.cpp:252-253
    sys_ = CudaGadiSystem(A, device=device, split=split if split.kind != "hss" else None)
    try:
        return sys_.solve(b, cfg, x0)
    finally:
        sys_.close()


def device_dot(x, y, p: Precision, device=0) -> float:
    """dot (kernels.cpp:84-90) on the device: rounded products, pairwise sum in p."""
    x, y = _f64(x), _f64(y)
    out = C.c_double()
    _check(lib().gadi_cuda_dot(device, int(p), _p(x), _p(y), len(x), C.byref(out)))
    return out.value


def device_norm2(x, p: Precision, device=0) -> float:
    """norm2 (kernels.cpp:71-82) with the pairwise sum on the device."""
    x = _f64(x)
    out = C.c_double()
    _check(lib().gadi_cuda_norm2(device, int(p), _p(x), len(x), C.byref(out)))
    return out.value


# ---------------------------------------------------------------- GPR
class GprModel:
    def __init__(self, handle):
        self._h = handle

    def params(self):
        v = [C.c_double() for _ in range(5)]
        _check(lib().gadi_gpr_params(self._h, *[C.byref(t) for t in v]))
        return dict(zip(("sigma_f2", "length", "sigma_n2", "lml", "target_mean"), [t.value for t in v]))

    def timings(self):
        """Device times (ms) of the fit, the inverse-factor formation and the last
        variance pass; the variance path taken ("tensor" = tcgen05, "fp64"); kernels launched."""
        f, i, v = C.c_double(), C.c_double(), C.c_double()
        path, n = C.c_int32(), C.c_int64()
        _check(lib().gadi_gpr_timings(self._h, C.byref(f), C.byref(i), C.byref(v), C.byref(path), C.byref(n)))
        return {"fit_ms": f.value, "inverse_ms": i.value, "variance_ms": v.value,
                "variance_path": {1: "tensor", 2: "fp64"}.get(path.value, "none"), "launches": n.value}

    def predict(self, sizes):
        sizes = _f64(sizes)
        mean = np.empty(len(sizes))
        sd = np.empty(len(sizes))
        _check(lib().gadi_gpr_predict(self._h, _p(sizes), len(sizes), _p(mean), _p(sd)))
        return mean, sd

    def predict_sharded(self, sizes, rank, world, group=None, gather=True):
        """predict_alpha over a rank's slice of the queries (they are independent: no
        data-path exchange); with gather=True every rank returns all (mean, sd), assembled
        in rank order over torch.distributed. Each query's result is the bits of predict()."""
        from .partition import gather_queries, query_shard
        sizes = _f64(sizes)
        lo, hi = query_shard(len(sizes), world, rank)
        mean, sd = self.predict(sizes[lo:hi]) if hi > lo else (np.empty(0), np.empty(0))
        if not gather:
            return mean, sd
        return gather_queries(mean, sd, len(sizes), group)

    def close(self):
        if self._h:
            lib().gadi_gpr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gpr_fit(sizes, alphas, fixed=None, sigma_n2=None, device=0) -> GprModel:
    """fit (gpr.cpp:109-149): grid search, or fixed (sigma_f2, length, sigma_n2)."""
    sizes, alphas = _f64(sizes), _f64(alphas)
    o = _GprOpts(0, 0.0, 0.0, 0.0, 0, device)
    if fixed is not None:
        o.fixed_hypers = 1
        o.sigma_f2, o.length, o.sigma_n2 = fixed
    elif sigma_n2 is not None:
        o.has_sigma_n2, o.sigma_n2 = 1, sigma_n2
    h = C.c_void_p()
    _check(lib().gadi_gpr_fit(_p(sizes), _p(alphas), len(sizes), C.byref(o), C.byref(h)))
    return GprModel(h)


# ---------------------------------------------------------------- training set (gpr.hpp:17-58,85-96)
@dataclass
class DichotomySettings:  # gpr.hpp:37-44
    alpha_lo: float = 1e-2
    alpha_hi: float = 1e2
    budget: int = 21
    train_xi: float = 1e-8
    max_outer: int = 1500
    inner: InnerSolverSpec = field(default_factory=InnerSolverSpec)

    def _c(self):
        return _Dichotomy(self.alpha_lo, self.alpha_hi, self.budget, self.train_xi, self.max_outer,
                          self.inner._c())


@dataclass
class TrainingPair:  # gpr.hpp:17-21
    size_n: int = 0
    alpha_opt: float = 0.0
    iters_at_opt: int = 0  # 0 marks a pseudo-pair added by retraining


@dataclass
class TrainingSet:  # gpr.hpp:23-26
    pairs: list = field(default_factory=list)  # sizes strictly increasing
    generation_precision: Precision = Precision.Single


def alpha_bisection(size_param: int, fmt: Precision, alpha_lo: float, alpha_hi: float, budget: int,
                    settings: Optional[DichotomySettings] = None, device: int = 0):
    """alpha_bisection (gpr.cpp:15-50) on the convdiff family (build_convdiff3d({n}), b = A*ones):
    budget log-spaced alphas, each a device solve with u_r = u = u_f = fmt, run concurrently.
    Returns (alpha, outer iterations); raises ParameterError / NoConvergentAlpha."""
    st = (settings or DichotomySettings())._c()
    a, it = C.c_double(), C.c_int32()
    _check(lib().gadi_alpha_bisection(int(size_param), int(fmt), alpha_lo, alpha_hi, int(budget), C.byref(st),
                                      device, C.byref(a), C.byref(it)))
    return a.value, it.value


def generate_training_set(size_params, fmt: Precision, settings: Optional[DichotomySettings] = None,
                          device: int = 0) -> TrainingSet:
    """generate_training_set (gpr.cpp:52-68): one (n^3, alpha_opt, iters) pair per size parameter."""
    st = settings or DichotomySettings()
    sp = np.ascontiguousarray(size_params, np.int64)
    k = len(sp)
    sn, al, it = np.zeros(k, np.int64), np.zeros(k), np.zeros(k, np.int32)
    _check(lib().gadi_generate_training_set(_p(sp, _i64p), k, int(fmt), C.byref(st._c()), device, _p(sn, _i64p),
                                            _p(al), _p(it, _i32p)))
    return TrainingSet([TrainingPair(int(a), float(b), int(c)) for a, b, c in zip(sn, al, it)], Precision(fmt))


def fit_training_set(ts: TrainingSet, sigma_n2=None, device=0) -> GprModel:
    """fit(ts) (gpr.cpp:109-149) on a TrainingSet."""
    return gpr_fit([p.size_n for p in ts.pairs], [p.alpha_opt for p in ts.pairs], sigma_n2=sigma_n2,
                   device=device)


def retrain_extend(model: GprModel, ts: TrainingSet, new_sizes) -> TrainingSet:
    """retrain_extend (gpr.cpp:171-186): append (size, predicted alpha, 0) pseudo-pairs for sizes
    not present, sorted by size."""
    out = TrainingSet(list(ts.pairs), ts.generation_precision)
    for s in new_sizes:
        if any(p.size_n == s for p in out.pairs):
            continue
        mean, _ = model.predict([float(s)])
        out.pairs.append(TrainingPair(int(s), float(mean[0]), 0))
    out.pairs.sort(key=lambda p: p.size_n)
    return out


_PNAME = {Precision.Half: "half", Precision.Single: "single", Precision.Double: "double"}


def write_training_csv(f, ts: TrainingSet):
    """write_training_csv (gpr.cpp:188-196): header n,alpha,iters,precision; %.17g alphas."""
    f.write("n,alpha,iters,precision\n")
    for p in ts.pairs:
        f.write(f"{p.size_n},{p.alpha_opt:.17g},{p.iters_at_opt},{_PNAME[ts.generation_precision]}\n")


def read_training_csv(f) -> TrainingSet:
    """read_training_csv (gpr.cpp:198-218)."""
    lines = f.read().splitlines()
    if not lines:
        raise GadiError("training csv: empty stream")  # IoError
    ts = TrainingSet()
    for line in lines[1:]:
        if not line:
            continue
        n, a, it, prec = line.split(",")[:4]
        ts.pairs.append(TrainingPair(int(n), float(a), int(it)))
        ts.generation_precision = {v: k for k, v in _PNAME.items()}[prec]
    return ts


# ---------------------------------------------------------------- MatrixMarket (sparse.hpp:75-76)
def read_matrix_market_file(path: str, device: int = 0) -> SparseMatrix:
    """read_matrix_market_file (matrix_market.cpp:22-62): host parse, from_triplets assembly on the
    device. Raises IoError / ContractViolation like the reference."""
    L = lib()
    h = C.c_void_p()
    _check(L.gadi_mm_read(os.fsencode(path), device, C.byref(h)))
    try:
        nr, nc, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        rp, ci, v = _i64p(), _i64p(), _f64p()
        _check(L.gadi_csr_view(h, C.byref(nr), C.byref(nc), C.byref(nnz), C.byref(rp), C.byref(ci), C.byref(v)))
        k = nnz.value
        arr = lambda ptr, n, dt: np.ctypeslib.as_array(ptr, (n,)).astype(dt, copy=True) if n else np.zeros(0, dt)
        return SparseMatrix(nr.value, nc.value, arr(rp, nr.value + 1, np.int64), arr(ci, k, np.int64),
                            arr(v, k, np.float64))
    finally:
        L.gadi_csr_destroy(h)


def write_matrix_market_file(path: str, A: SparseMatrix):
    """write_matrix_market_file (matrix_market.cpp:64-86)."""
    _check(lib().gadi_mm_write(os.fsencode(path), A.n_rows, A.n_cols, _p(A.row_ptr, _i64p), _p(A.col_idx, _i64p),
                               _p(A.values)))


# ---------------------------------------------------------------- Sylvester GADI-AB (problems.hpp:34-89)
def tridiag(n: int, sub: float, diag: float, sup: float) -> SparseMatrix:
    """SparseMatrix::tridiag (sparse.cpp:76-85); zero bands are not stored."""
    rp, ci, v = [0], [], []
    for i in range(n):
        for c, x in ((i - 1, sub), (i, diag), (i + 1, sup)):
            if 0 <= c < n and x != 0.0:
                ci.append(c)
                v.append(x)
        rp.append(len(ci))
    return SparseMatrix(n, n, rp, ci, v)


@dataclass
class SylvesterProblem:  # problems.hpp:39-44
    A: SparseMatrix
    B: SparseMatrix
    C_rhs: np.ndarray    # A X + X B + C = 0
    X_exact: np.ndarray


def build_sylvester(n: int, r: float = 1.0) -> SylvesterProblem:
    """build_sylvester (problems.cpp:45-66): A = B = Tridiag(-1-r, 2+shift, -1+r),
    shift = 100/(n+1)^2, X = ones, C = -(A X + X B) from row/column sums."""
    if n < 2:
        raise ContractViolation("sylvester: n >= 2 required")
    if not r > 0.0:
        raise ContractViolation("sylvester: r > 0 required")
    sh = 100.0 / ((float(n) + 1.0) * (float(n) + 1.0))
    A = tridiag(n, -1.0 - r, 2.0 + sh, -1.0 + r)
    row, col = np.zeros(n), np.zeros(n)
    for i in range(n):
        for k in range(A.row_ptr[i], A.row_ptr[i + 1]):
            row[i] += A.values[k]
            col[A.col_idx[k]] += A.values[k]
    C_rhs = -(row[:, None] + col[None, :])
    return SylvesterProblem(A, A, C_rhs, np.ones((n, n)))


@dataclass
class SylvesterResult:  # problems.hpp:86-89
    X: np.ndarray
    report: SolveReport


def gadi_ab_solve(prob: SylvesterProblem, cfg: GadiConfig, device: int = 0) -> SylvesterResult:
    """gadi_ab_solve (sylvester.cpp:122-133): run_gadi_ir over the SylvesterOperator on the device
    (G = -C, x0 = zeros or ones)."""
    L = lib()
    m, n = prob.A.n_rows, prob.B.n_rows
    G = np.ascontiguousarray((-np.asarray(prob.C_rhs, np.float64)).T).reshape(-1)  # column-major vec
    h = C.c_void_p()
    A, B = prob.A, prob.B
    _check(L.gadi_sylv_create(m, _p(A.row_ptr, _i64p), _p(A.col_idx, _i64p), _p(A.values), n,
                              _p(B.row_ptr, _i64p), _p(B.col_idx, _i64p), _p(B.values), _p(G), device,
                              C.byref(h)))
    try:
        x = np.empty(m * n)
        rep = _Report()
        c = cfg._c()
        _check(L.gadi_sylv_solve(h, C.byref(c), None, _p(x), C.byref(rep)))
        hist = np.empty(max(rep.history_len, 1))
        L.gadi_sylv_history(h, _p(hist), len(hist))
        r = SolveReport(status=SolveStatus(rep.status), outer_iters=rep.outer_iters,
                        rel_residual_history=hist[:rep.history_len].copy(), final_rres=rep.final_rres,
                        inner_iter_totals=rep.inner_iter_totals, inner_stagnations=rep.inner_stagnations,
                        solve_ms=rep.solve_ms, launches=rep.launches)
        return SylvesterResult(x.reshape(n, m).T.copy(), r)
    finally:
        L.gadi_sylv_destroy(h)
