"""Golden solves with EXPLICIT splittings (tests/golden/explicit_split.npz).

Runs the reference's gadi_ir_solve(A, b, explicit_splitting(A, M, N), cfg)
(splitting.cpp:22-35, solver.cpp:250-258; oracle/_ref/libgadi_ref.so) on
build_convdiff3d(6) with three non-HSS splittings and stores M, N and the
results; the CPU test pins the oracle restatement to them and the GPU test
compares the device path (gadi_cuda_set_split) with them bit for bit.

    make -f oracle/Makefile.ref && python tests/golden/make_golden_split.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import CG, CSR, DOUBLE, GMRES, HALF, SINGLE, Config, Oracle, Reference  # noqa: E402


def weighted(A, wl, wd, wu):
    """M = wl*L + wd*D + wu*U (entries with weight 0 are absent), N = A - M
    (entries with weight 1 are absent)."""
    parts = [([0], [], []), ([0], [], [])]
    for i in range(A.n):
        for k in range(A.rp[i], A.rp[i + 1]):
            c, a = int(A.ci[k]), float(A.v[k])
            w = wd if c == i else (wl if c < i else wu)
            m = a * w
            if w != 0.0:
                parts[0][1].append(c)
                parts[0][2].append(m)
            if w != 1.0:
                parts[1][1].append(c)
                parts[1][2].append(a - m)
        for p in parts:
            p[0].append(len(p[1]))
    return [CSR(A.n, *p) for p in parts]


def splits(o, A):
    """name -> (M, N)."""
    out = {}
    # 1. three quarters of the symmetric part (H stays SPD: CG applies), N = the skew part plus the rest
    Mh, Nh = o.regularize(A, 0.0)  # M, N of the HSS split on the union pattern
    out["symshift"] = (CSR(A.n, Mh.rp, Mh.ci, 0.75 * Mh.v), CSR(A.n, Nh.rp, Nh.ci, Nh.v + 0.25 * Mh.v))
    # 2. Gauss-Seidel like: M = L + D/2 + U/4 (nonsymmetric)
    out["tri"] = tuple(weighted(A, 1.0, 0.5, 0.25))
    # 3. N without any diagonal entry (shift_diagonal inserts it), M carries the diagonal
    out["nodiag"] = tuple(weighted(A, 0.5, 1.0, 0.5))
    return out


CASES = [  # (split, u_r, kwargs)
    ("symshift", SINGLE, dict(method=CG, tol_epsilon=1e-10, max_inner_iters=40, alpha=0.8, xi=1e-14)),
    ("symshift", HALF, dict(method=CG, tol_epsilon=1e-4, max_inner_iters=40, alpha=0.8, xi=1e-6,
                            max_outer_iters=300)),
    ("tri", DOUBLE, dict(method=GMRES, tol_epsilon=1e-10, max_inner_iters=40, alpha=0.8, xi=1e-12,
                         max_outer_iters=3000)),
    ("tri", HALF, dict(method=0, alpha=0.8, xi=1e-8)),
    ("tri", SINGLE, dict(method=0, alpha=0.5, xi=1e-12)),
    ("nodiag", SINGLE, dict(method=GMRES, tol_epsilon=1e-8, max_inner_iters=30, restart=10, alpha=4.0, xi=1e-12,
                            max_outer_iters=400)),
    ("nodiag", DOUBLE, dict(method=0, alpha=4.0, xi=1e-20, max_outer_iters=400)),
]


def main():
    R, o = Reference(), Oracle()
    A = o.convdiff(6)
    _, b = o.make_rhs(A, 3, -1.0, 1.0)
    out = {"b": b}
    sp = splits(o, A)
    for nm, (M, N) in sp.items():
        for t, X in (("M", M), ("N", N)):
            out[f"{nm}_{t}_rp"], out[f"{nm}_{t}_ci"], out[f"{nm}_{t}_v"] = X.rp, X.ci, X.v
    for i, (nm, ur, kw) in enumerate(CASES):
        M, N = sp[nm]
        x, rep, hist = R.solve_split(A, M, N, b, Config.make(u_r=ur, **kw))
        out[f"case{i}_x"], out[f"case{i}_hist"] = x, hist
        out[f"case{i}_info"] = np.array([rep.status, rep.outer_iters, rep.inner_iter_totals, rep.inner_stagnations])
        print(i, nm, ur, rep.status, rep.outer_iters, rep.inner_iter_totals, hist[-1])
    path = os.path.join(HERE, "explicit_split.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path))


if __name__ == "__main__":
    main()
