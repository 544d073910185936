import sys, ctypes as C, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2501_04229_b200 as g
from oracle import *
orc = Oracle()
L = C.CDLL('/root/repo/oracle/_ref/libgadi_ref_cuda.so')
f64p = C.POINTER(C.c_double)
L.refcuda_solve_stencil.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double, f64p, C.POINTER(Config), f64p, f64p, C.c_int, C.POINTER(Report)]
for n, ur, alpha in ((16, 1, 0.1), (8, 0, 0.5), (8, 1, 0.2)):
    S = g.build_convdiff3d(n); A = orc.convdiff(n, S.t1, S.t2, S.t3)
    _, b = orc.make_rhs(A, 0, 0.0, 1.0)
    cfg = Config.make(alpha=alpha, xi=1e-20, u_r=ur, method=CG, tol_epsilon=1e-12, max_inner_iters=50)
    x = np.zeros(A.n); hist = np.zeros(10000); rep = Report()
    p = lambda a: a.ctypes.data_as(f64p)
    rc = L.refcuda_solve_stencil(n, S.t1, S.t2, S.t3, p(b), C.byref(cfg), p(x), p(hist), 10000, C.byref(rep))
    wx, wrep, wh = orc.solve(A, b, cfg)
    print(n, ur, rc, rep.outer_iters, wrep.outer_iters, rep.inner_iter_totals, wrep.inner_iter_totals, np.abs(x - wx).max(), np.abs(hist[:rep.history_len] - wh).max())
