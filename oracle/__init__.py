"""ctypes bindings for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two libraries:
  * ``oracle/liboracle.so`` — the C restatement of the reference hot path
    (``oracle/gadi_oracle.c``); always available (``make -C oracle``).
  * ``oracle/_ref/libgadi_ref.so`` — the reference itself, compiled from
    /root/reference by ``oracle/Makefile.ref``; available where it was built.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline leg may
import this package; the product (``paper_2501_04229_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_ORACLE = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libgadi_ref.so")

HALF, SINGLE, DOUBLE = 0, 1, 2
LU_DIRECT, CG, GMRES = 0, 1, 2

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


class InnerSpec(C.Structure):
    _fields_ = [("method", C.c_int32), ("tol_epsilon", C.c_double),
                ("max_inner_iters", C.c_int32), ("restart", C.c_int32)]


class Config(C.Structure):
    """gadi_config (include/gadi_cuda.h) = GadiConfig (solver.hpp:17-38)."""
    _fields_ = [("alpha", C.c_double), ("omega", C.c_double), ("xi", C.c_double),
                ("u_r", C.c_int32), ("u", C.c_int32), ("u_f", C.c_int32),
                ("inner", InnerSpec), ("max_outer_iters", C.c_int32),
                ("divergence_factor", C.c_double), ("stall_window", C.c_int32),
                ("ones_start", C.c_int32), ("residual_scaling", C.c_int32),
                ("accum", C.c_int32)]

    @classmethod
    def make(cls, **kw):
        c = cls(alpha=1.0, omega=1.0, xi=0.0, u_r=DOUBLE, u=DOUBLE, u_f=DOUBLE,
                inner=InnerSpec(LU_DIRECT, 1e-2, 1000, 30), max_outer_iters=20000,
                divergence_factor=1e6, stall_window=0, ones_start=0, residual_scaling=1,
                accum=0)
        for k, v in kw.items():
            if k in ("method", "tol_epsilon", "max_inner_iters", "restart"):
                setattr(c.inner, k, v)
            else:
                setattr(c, k, v)
        return c


class Dichotomy(C.Structure):  # gadi_dichotomy = DichotomySettings (gpr.hpp:37-44)
    _fields_ = [("alpha_lo", C.c_double), ("alpha_hi", C.c_double), ("budget", C.c_int32),
                ("train_xi", C.c_double), ("max_outer", C.c_int32), ("inner", InnerSpec)]

    @classmethod
    def make(cls, **kw):
        d = cls(1e-2, 1e2, 21, 1e-8, 1500, InnerSpec(LU_DIRECT, 1e-2, 1000, 30))
        for k, v in kw.items():
            if k in ("method", "tol_epsilon", "max_inner_iters", "restart"):
                setattr(d.inner, k, v)
            else:
                setattr(d, k, v)
        return d


class Report(C.Structure):
    _fields_ = [("status", C.c_int32), ("outer_iters", C.c_int32), ("final_rres", C.c_double),
                ("inner_iter_totals", C.c_int64), ("inner_stagnations", C.c_int32),
                ("history_len", C.c_int32), ("h_iters", C.c_int64), ("s_iters", C.c_int64),
                ("solve_ms", C.c_double), ("h_ms", C.c_double), ("s_ms", C.c_double),
                ("outer_ms", C.c_double), ("h2d_bytes", C.c_double), ("d2h_bytes", C.c_double),
                ("e2e_ms", C.c_double), ("launches", C.c_int64)]


class GprOpts(C.Structure):
    _fields_ = [("fixed_hypers", C.c_int32), ("sigma_f2", C.c_double), ("length", C.c_double),
                ("sigma_n2", C.c_double), ("has_sigma_n2", C.c_int32), ("device", C.c_int32)]


def _p(a, t=_f64p):
    return None if a is None else a.ctypes.data_as(t)


def build_oracle():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class CSR:
    """Reference SparseMatrix layout (sparse.hpp:17-65): int64 rp/ci, fp64 v."""

    def __init__(self, n, rp, ci, v):
        self.n = int(n)
        self.rp = np.ascontiguousarray(rp, dtype=np.int64)
        self.ci = np.ascontiguousarray(ci, dtype=np.int64)
        self.v = np.ascontiguousarray(v, dtype=np.float64)

    @property
    def nnz(self):
        return int(self.rp[-1])


class _OrcCsr(C.Structure):
    _fields_ = [("n", C.c_int64), ("rp", _i64p), ("ci", _i64p), ("v", _f64p)]


def _oc(A: CSR):
    return _OrcCsr(A.n, _p(A.rp, _i64p), _p(A.ci, _i64p), _p(A.v))


class Oracle:
    """The C restatement (oracle/gadi_oracle.c)."""

    def __init__(self, path=LIB_ORACLE):
        if not os.path.exists(path):
            build_oracle()
        L = self.L = C.CDLL(path)
        L.orc_round.restype = C.c_double
        L.orc_round.argtypes = [C.c_double, C.c_int]
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_uniform.restype = C.c_double
        L.orc_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double]
        L.orc_convdiff_csr.restype = C.c_int64
        L.orc_convdiff_csr.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double, _i64p, _i64p, _f64p]
        L.orc_band_csr.restype = C.c_int64
        L.orc_band_csr.argtypes = [C.c_int64, C.c_int32, C.c_int64, C.c_uint64, _i64p, _i64p, _f64p]
        L.orc_make_rhs.restype = None
        L.orc_make_rhs.argtypes = [C.POINTER(_OrcCsr), C.c_uint64, C.c_double, C.c_double, _f64p, _f64p]
        L.orc_matvec.argtypes = [C.POINTER(_OrcCsr), _f64p, C.c_int, _f64p]
        L.orc_residual.argtypes = [C.POINTER(_OrcCsr), _f64p, _f64p, C.c_int, C.c_int, _f64p]
        for f in ("orc_dot",):
            getattr(L, f).restype = C.c_double
        L.orc_dot.argtypes = [_f64p, _f64p, C.c_int64, C.c_int]
        L.orc_norm2.restype = C.c_double
        L.orc_norm2.argtypes = [_f64p, C.c_int64, C.c_int]
        L.orc_norm2_64.restype = C.c_double
        L.orc_norm2_64.argtypes = [_f64p, C.c_int64]
        L.orc_axpy.argtypes = [C.c_double, _f64p, _f64p, C.c_int64, C.c_int, _f64p]
        L.orc_scale.argtypes = [C.c_double, _f64p, C.c_int64, C.c_int, _f64p]
        L.orc_regularize.restype = C.c_int64
        L.orc_regularize.argtypes = [C.POINTER(_OrcCsr), C.c_double, _i64p, _i64p, _f64p, _f64p]
        L.orc_krylov.argtypes = [C.POINTER(_OrcCsr), _f64p, C.c_int, C.c_double, C.c_int, C.c_int,
                                 C.c_int, C.c_double, _f64p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.orc_krylov_af.argtypes = [C.POINTER(_OrcCsr), _f64p, C.c_int, C.c_double, C.c_int, C.c_int,
                                    C.c_int, C.c_int, C.c_double, _f64p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.orc_alpha_bisection.argtypes = [C.c_int64, C.c_int, C.c_double, C.c_double, C.c_int,
                                           C.POINTER(Dichotomy), _f64p, C.POINTER(C.c_int)]
        L.orc_lu_solve.argtypes = [C.POINTER(_OrcCsr), _f64p, C.c_int, _f64p]
        L.orc_solve.argtypes = [C.POINTER(_OrcCsr), _f64p, _f64p, C.POINTER(Config), _f64p, _f64p,
                                C.c_int, C.POINTER(Report)]
        L.orc_solve_split.argtypes = [C.POINTER(_OrcCsr), C.POINTER(_OrcCsr), C.POINTER(_OrcCsr), _f64p, _f64p,
                                      C.POINTER(Config), _f64p, _f64p, C.c_int, C.POINTER(Report)]
        L.orc_gpr.argtypes = [_f64p, _f64p, C.c_int, C.POINTER(GprOpts), _f64p, C.c_int, _f64p,
                              _f64p, _f64p]

    # ---- rounding / rng
    def round(self, x, p):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return np.array([self.L.orc_round(float(v), p) for v in x.ravel()]).reshape(x.shape)

    def uniform(self, seed, n, lo, hi):
        return np.array([self.L.orc_uniform(seed, i, lo, hi) for i in range(n)])

    # ---- generators
    def convdiff(self, n, t1=6.0, t2=None, t3=None, r=None):
        if r is None:
            r = 1.0 / (2.0 * n + 2.0)
        if t2 is None:
            t2 = -1.0 - r
        if t3 is None:
            t3 = -1.0 + r
        N = n ** 3
        rp = np.zeros(N + 1, np.int64)
        ci = np.zeros(7 * N, np.int64)
        v = np.zeros(7 * N, np.float64)
        nnz = self.L.orc_convdiff_csr(n, t1, t2, t3, _p(rp, _i64p), _p(ci, _i64p), _p(v))
        return CSR(N, rp, ci[:nnz], v[:nnz])

    def band(self, N, k_off=26, band=4096, seed=2):
        rp = np.zeros(N + 1, np.int64)
        ci = np.zeros(N * (k_off + 1), np.int64)
        v = np.zeros(N * (k_off + 1), np.float64)
        nnz = self.L.orc_band_csr(N, k_off, band, seed, _p(rp, _i64p), _p(ci, _i64p), _p(v))
        return CSR(N, rp, ci[:nnz], v[:nnz])

    def make_rhs(self, A: CSR, seed, lo, hi):
        x = np.zeros(A.n)
        b = np.zeros(A.n)
        oc = _oc(A)
        self.L.orc_make_rhs(C.byref(oc), seed, lo, hi, _p(x), _p(b))
        return x, b

    # ---- kernels
    def matvec(self, A, x, p):
        y = np.zeros(A.n)
        oc = _oc(A)
        self.L.orc_matvec(C.byref(oc), _p(np.ascontiguousarray(x, np.float64)), p, _p(y))
        return y

    def residual(self, A, x, b, uf, ur):
        s = np.zeros(A.n)
        oc = _oc(A)
        self.L.orc_residual(C.byref(oc), _p(np.ascontiguousarray(x, np.float64)),
                            _p(np.ascontiguousarray(b, np.float64)), uf, ur, _p(s))
        return s

    def dot(self, x, y, p):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        return self.L.orc_dot(_p(x), _p(y), len(x), p)

    def norm2(self, x, p):
        x = np.ascontiguousarray(x, np.float64)
        return self.L.orc_norm2(_p(x), len(x), p)

    def norm2_64(self, x):
        x = np.ascontiguousarray(x, np.float64)
        return self.L.orc_norm2_64(_p(x), len(x))

    def axpy(self, a, x, y, p):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        z = np.zeros(len(x))
        self.L.orc_axpy(a, _p(x), _p(y), len(x), p, _p(z))
        return z

    def scale(self, a, x, p):
        x = np.ascontiguousarray(x, np.float64)
        z = np.zeros(len(x))
        self.L.orc_scale(a, _p(x), len(x), p, _p(z))
        return z

    def regularize(self, A: CSR, alpha):
        oc = _oc(A)
        nnz = self.L.orc_regularize(C.byref(oc), alpha, None, None, None, None)
        rp = np.zeros(A.n + 1, np.int64)
        ci = np.zeros(nnz, np.int64)
        vh = np.zeros(nnz)
        vs = np.zeros(nnz)
        self.L.orc_regularize(C.byref(oc), alpha, _p(rp, _i64p), _p(ci, _i64p), _p(vh), _p(vs))
        return CSR(A.n, rp, ci, vh), CSR(A.n, rp, ci, vs)

    def krylov(self, M: CSR, rhs, method, eps, max_inner, restart, fmt, stop_norm, af=None):
        """af: arithmetic format (None = fmt, the reference); SINGLE over HALF
        storage restates the device's GADI_ACCUM_FP32 inner mode."""
        rhs = np.ascontiguousarray(rhs, np.float64)
        x = np.zeros(M.n)
        it, st = C.c_int(), C.c_int()
        oc = _oc(M)
        self.L.orc_krylov_af(C.byref(oc), _p(rhs), method, eps, max_inner, restart, fmt,
                             fmt if af is None else af, stop_norm, _p(x), C.byref(it), C.byref(st))
        return x, it.value, st.value

    def alpha_bisection(self, n, fmt, lo, hi, budget, st):
        """(alpha, iters), or raise on the reference's exceptions (rc -2 / -11)."""
        a, it = C.c_double(), C.c_int()
        rc = self.L.orc_alpha_bisection(n, fmt, lo, hi, budget, C.byref(st), C.byref(a), C.byref(it))
        if rc != 0:
            raise ValueError(rc)
        return a.value, it.value

    def lu_solve(self, M: CSR, rhs, fmt):
        """BandLU factor + solve of M in fmt (band_lu.cpp); returns (x, status)
        with status 0, 4 (SingularInPrecision) or 3 (OverflowDetected)."""
        rhs = np.ascontiguousarray(rhs, np.float64)
        x = np.zeros(M.n)
        oc = _oc(M)
        st = self.L.orc_lu_solve(C.byref(oc), _p(rhs), fmt, _p(x))
        return x, st

    def solve(self, A: CSR, b, cfg: Config, x0=None, cap=100000, split=None):
        """split = (M, N): explicit_splitting(A, M, N) (splitting.cpp:22-35); None: hss_split."""
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(A.n)
        hist = np.zeros(cap)
        rep = Report()
        oc = _oc(A)
        x0a = None if x0 is None else np.ascontiguousarray(x0, np.float64)
        if split is None:
            rc = self.L.orc_solve(C.byref(oc), _p(b), _p(x0a), C.byref(cfg), _p(x), _p(hist), cap,
                                  C.byref(rep))
        else:
            om, on = _oc(split[0]), _oc(split[1])
            rc = self.L.orc_solve_split(C.byref(oc), C.byref(om), C.byref(on), _p(b), _p(x0a), C.byref(cfg),
                                        _p(x), _p(hist), cap, C.byref(rep))
        if rc != 0:
            raise ValueError(f"orc_solve rc={rc}")
        return x, rep, hist[: min(rep.history_len, cap)].copy()

    def gpr(self, sizes, alphas, qsizes, fixed=None, sigma_n2=None):
        sizes = np.ascontiguousarray(sizes, np.float64)
        alphas = np.ascontiguousarray(alphas, np.float64)
        qsizes = np.ascontiguousarray(qsizes, np.float64)
        o = GprOpts(0, 0.0, 0.0, 0.0, 0, 0)
        if fixed is not None:
            o.fixed_hypers = 1
            o.sigma_f2, o.length, o.sigma_n2 = fixed
        elif sigma_n2 is not None:
            o.has_sigma_n2, o.sigma_n2 = 1, sigma_n2
        mean = np.zeros(len(qsizes))
        sd = np.zeros(len(qsizes))
        params = np.zeros(5)
        rc = self.L.orc_gpr(_p(sizes), _p(alphas), len(sizes), C.byref(o), _p(qsizes), len(qsizes),
                            _p(mean), _p(sd), _p(params))
        if rc != 0:
            raise ValueError(f"orc_gpr rc={rc}")
        return mean, sd, params


class Reference:
    """The reference itself (oracle/_ref/libgadi_ref.so, built from /root/reference)."""

    @staticmethod
    def available(path=LIB_REF):
        return os.path.exists(path)

    def __init__(self, path=LIB_REF):
        L = self.L = C.CDLL(path)
        L.ref_build_convdiff.argtypes = [C.c_int64, _i64p, _i64p, _f64p, _f64p]
        L.ref_round.argtypes = [_f64p, C.c_int64, C.c_int, _f64p]
        L.ref_matvec.argtypes = [C.c_int64, _i64p, _i64p, _f64p, _f64p, C.c_int, _f64p]
        L.ref_residual.argtypes = [C.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p, C.c_int, C.c_int, _f64p]
        L.ref_dot.restype = C.c_double
        L.ref_dot.argtypes = [_f64p, _f64p, C.c_int64, C.c_int]
        L.ref_norm2.restype = C.c_double
        L.ref_norm2.argtypes = [_f64p, C.c_int64, C.c_int]
        L.ref_norm2_64.restype = C.c_double
        L.ref_norm2_64.argtypes = [_f64p, C.c_int64]
        L.ref_axpy.argtypes = [C.c_double, _f64p, _f64p, C.c_int64, C.c_int, _f64p]
        L.ref_scale.argtypes = [C.c_double, _f64p, C.c_int64, C.c_int, _f64p]
        L.ref_regularize.restype = C.c_int64
        L.ref_regularize.argtypes = [C.c_int64, _i64p, _i64p, _f64p, C.c_double, C.c_double, _i64p,
                                     _i64p, _f64p, _f64p]
        L.ref_krylov.argtypes = [C.c_int64, _i64p, _i64p, _f64p, _f64p, C.c_int, C.c_double, C.c_int,
                                 C.c_int, C.c_int, C.c_double, _f64p, C.POINTER(C.c_int),
                                 C.POINTER(C.c_int)]
        L.ref_alpha_bisection.argtypes = [C.c_int64, C.c_int, C.c_double, C.c_double, C.c_int,
                                           C.POINTER(Dichotomy), _f64p, C.POINTER(C.c_int)]
        L.ref_mm_read.restype = C.c_int64
        L.ref_mm_read.argtypes = [C.c_char_p, _i64p, _i64p, _i64p, _i64p, _f64p]
        L.ref_sylvester_solve.argtypes = [C.c_int64, C.c_double, C.POINTER(Config), _f64p, _f64p, C.c_int,
                                           C.POINTER(Report)]
        L.ref_lu_solve.argtypes = [C.c_int64, _i64p, _i64p, _f64p, _f64p, C.c_int, _f64p]
        L.ref_solve.argtypes = [C.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p, C.POINTER(Config), _f64p,
                                _f64p, C.c_int, C.POINTER(Report)]
        L.ref_reference_solve.argtypes = [C.c_int64, _i64p, _i64p, _f64p, _f64p, C.c_double, C.c_double,
                                          C.c_double, C.c_int, _f64p, C.POINTER(C.c_int),
                                          C.POINTER(C.c_int)]
        L.ref_solve_split.argtypes = [C.c_int64, _i64p, _i64p, _f64p, _i64p, _i64p, _f64p, _i64p, _i64p, _f64p,
                                      _f64p, C.POINTER(Config), _f64p, _f64p, C.c_int, C.POINTER(Report)]
        L.ref_solve_steps_timed.argtypes = [C.c_int64, _i64p, _i64p, _f64p, _f64p, C.POINTER(Config), C.c_int,
                                            C.c_int, _f64p, C.POINTER(C.c_int)]
        L.ref_gpr.argtypes = [_i64p, _f64p, C.c_int, C.c_int, C.c_double, _i64p, C.c_int, _f64p, _f64p,
                              _f64p]

    @staticmethod
    def _a(A):
        return (A.n, _p(A.rp, _i64p), _p(A.ci, _i64p), _p(A.v))

    def convdiff(self, n):
        N = n ** 3
        nnz = 7 * n ** 3 - 6 * n ** 2
        rp = np.zeros(N + 1, np.int64)
        ci = np.zeros(nnz, np.int64)
        v = np.zeros(nnz)
        b = np.zeros(N)
        assert self.L.ref_build_convdiff(n, _p(rp, _i64p), _p(ci, _i64p), _p(v), _p(b)) == 0
        return CSR(N, rp, ci, v), b

    def round(self, x, p):
        x = np.ascontiguousarray(x, np.float64)
        o = np.zeros_like(x)
        self.L.ref_round(_p(x), x.size, p, _p(o))
        return o

    def matvec(self, A, x, p):
        y = np.zeros(A.n)
        assert self.L.ref_matvec(*self._a(A), _p(np.ascontiguousarray(x, np.float64)), p, _p(y)) == 0
        return y

    def residual(self, A, x, b, uf, ur):
        s = np.zeros(A.n)
        assert self.L.ref_residual(*self._a(A), _p(np.ascontiguousarray(x, np.float64)),
                                   _p(np.ascontiguousarray(b, np.float64)), uf, ur, _p(s)) == 0
        return s

    def dot(self, x, y, p):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        return self.L.ref_dot(_p(x), _p(y), len(x), p)

    def norm2(self, x, p):
        x = np.ascontiguousarray(x, np.float64)
        return self.L.ref_norm2(_p(x), len(x), p)

    def norm2_64(self, x):
        x = np.ascontiguousarray(x, np.float64)
        return self.L.ref_norm2_64(_p(x), len(x))

    def axpy(self, a, x, y, p):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        z = np.zeros(len(x))
        self.L.ref_axpy(a, _p(x), _p(y), len(x), p, _p(z))
        return z

    def scale(self, a, x, p):
        x = np.ascontiguousarray(x, np.float64)
        z = np.zeros(len(x))
        self.L.ref_scale(a, _p(x), len(x), p, _p(z))
        return z

    def regularize(self, A, alpha, omega=1.0):
        nnz = self.L.ref_regularize(*self._a(A), alpha, omega, None, None, None, None)
        assert nnz >= 0, nnz
        rp = np.zeros(A.n + 1, np.int64)
        ci = np.zeros(nnz, np.int64)
        vh = np.zeros(nnz)
        vs = np.zeros(nnz)
        self.L.ref_regularize(*self._a(A), alpha, omega, _p(rp, _i64p), _p(ci, _i64p), _p(vh), _p(vs))
        return CSR(A.n, rp, ci, vh), CSR(A.n, rp, ci, vs)

    def krylov(self, M, rhs, method, eps, max_inner, restart, fmt, stop_norm):
        rhs = np.ascontiguousarray(rhs, np.float64)
        x = np.zeros(M.n)
        it, st = C.c_int(), C.c_int()
        assert self.L.ref_krylov(*self._a(M), _p(rhs), method, eps, max_inner, restart, fmt, stop_norm,
                                 _p(x), C.byref(it), C.byref(st)) == 0
        return x, it.value, st.value

    def alpha_bisection(self, n, fmt, lo, hi, budget, st):
        """(alpha, iters), or raise on the reference's exceptions (rc -2 / -11)."""
        a, it = C.c_double(), C.c_int()
        rc = self.L.ref_alpha_bisection(n, fmt, lo, hi, budget, C.byref(st), C.byref(a), C.byref(it))
        if rc != 0:
            raise ValueError(rc)
        return a.value, it.value

    def mm_read(self, path):
        """read_matrix_market_file: (n_rows, n_cols, rp, ci, v), or the error code (int)."""
        nr, nc = C.c_int64(), C.c_int64()
        nnz = self.L.ref_mm_read(path.encode(), C.byref(nr), C.byref(nc), None, None, None)
        if nnz < 0:
            return int(nnz)
        rp, ci, v = np.zeros(nr.value + 1, np.int64), np.zeros(nnz, np.int64), np.zeros(nnz)
        self.L.ref_mm_read(path.encode(), C.byref(nr), C.byref(nc), _p(rp, _i64p), _p(ci, _i64p), _p(v))
        return nr.value, nc.value, rp, ci, v

    def sylvester_solve(self, n, r, cfg, cap=100000):
        """gadi_ab_solve(build_sylvester({n, r}), cfg): (X column-major vec, report, history)."""
        X = np.zeros(n * n)
        hist = np.zeros(cap)
        rep = Report()
        assert self.L.ref_sylvester_solve(n, r, C.byref(cfg), _p(X), _p(hist), cap, C.byref(rep)) == 0
        return X, rep, hist[: min(rep.history_len, cap)].copy()

    def lu_solve(self, M, rhs, fmt):
        rhs = np.ascontiguousarray(rhs, np.float64)
        x = np.zeros(M.n)
        st = self.L.ref_lu_solve(*self._a(M), _p(rhs), fmt, _p(x))
        assert st >= 0, st
        return x, st

    def solve(self, A, b, cfg, x0=None, cap=100000):
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(A.n)
        hist = np.zeros(cap)
        rep = Report()
        x0a = None if x0 is None else np.ascontiguousarray(x0, np.float64)
        rc = self.L.ref_solve(*self._a(A), _p(b), _p(x0a), C.byref(cfg), _p(x), _p(hist), cap,
                              C.byref(rep))
        if rc != 0:
            raise ValueError(f"ref_solve rc={rc}")
        return x, rep, hist[: min(rep.history_len, cap)].copy()

    def solve_split(self, A, M, N, b, cfg, cap=100000):
        """gadi_ir_solve(A, b, explicit_splitting(A, M, N), cfg)."""
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(A.n)
        hist = np.zeros(cap)
        rep = Report()
        rc = self.L.ref_solve_split(*self._a(A), *self._a(M)[1:], *self._a(N)[1:], _p(b), C.byref(cfg), _p(x),
                                    _p(hist), cap, C.byref(rep))
        if rc != 0:
            raise ValueError(rc)
        return x, rep, hist[: min(rep.history_len, cap)].copy()

    def solve_steps_timed(self, A, b, cfg, k1, k2):
        """(split_s, solve_k1_s, solve_k2_s, outer_k1, outer_k2): the split once, then
        gadi_ir_solve capped at k1 and at k2 outer steps (bench.py's CPU baseline)."""
        b = np.ascontiguousarray(b, np.float64)
        t = np.zeros(3)
        it = (C.c_int * 2)()
        rc = self.L.ref_solve_steps_timed(*self._a(A), _p(b), C.byref(cfg), k1, k2, _p(t), it)
        if rc != 0:
            raise ValueError(f"ref_solve_steps_timed rc={rc}")
        return t[0], t[1], t[2], it[0], it[1]

    def gpr(self, sizes, alphas, qsizes, sigma_n2=None):
        sizes = np.ascontiguousarray(sizes, np.int64)
        alphas = np.ascontiguousarray(alphas, np.float64)
        qsizes = np.ascontiguousarray(qsizes, np.int64)
        mean = np.zeros(len(qsizes))
        sd = np.zeros(len(qsizes))
        params = np.zeros(4)
        rc = self.L.ref_gpr(_p(sizes, _i64p), _p(alphas), len(sizes), int(sigma_n2 is not None),
                            0.0 if sigma_n2 is None else sigma_n2, _p(qsizes, _i64p), len(qsizes),
                            _p(mean), _p(sd), _p(params))
        if rc != 0:
            raise ValueError(f"ref_gpr rc={rc}")
        return mean, sd, params
