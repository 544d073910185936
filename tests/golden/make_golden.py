"""Generate the golden vectors in tests/golden/ from the REFERENCE itself.

Runs the reference's own code (oracle/_ref/libgadi_ref.so, compiled from
/root/reference/proj/core by oracle/Makefile.ref) on small seeded inputs and
stores inputs + outputs as .npz fixtures. The CPU tests pin the oracle
restatement to these files bit for bit, and the GPU tests compare the device
path with them, so neither needs /root/reference at run time.

    make -f oracle/Makefile.ref && python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import CG, CSR, DOUBLE, GMRES, HALF, SINGLE, Config, Dichotomy, Oracle, Reference  # noqa: E402

LU = 0  # InnerMethod::LuDirect


def main():
    R = Reference()
    o = Oracle()  # used only for the seeded generators (themselves pinned below)
    out = {}

    # 1. rounding KATs: all 65,536 binary16 encodings re-rounded, and random doubles
    enc = np.arange(65536, dtype=np.uint16).view(np.float16).astype(np.float64)
    enc = enc[np.isfinite(enc)]
    rng = np.random.default_rng(20250104)
    rand = rng.standard_normal(20000) * 10.0 ** rng.integers(-9, 6, 20000)
    edge = np.array([65504.0, 65519.999, 65520.0, 2.0 ** -24, 2.0 ** -25, 1.5 * 2.0 ** -25, 3 * 2.0 ** -26,
                     -0.0, 0.0, 1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11, 2.0 ** -14 * (1 - 2.0 ** -11)])
    xs = np.concatenate([enc, rand, edge])
    out["round_x"] = xs
    for p, nm in ((HALF, "half"), (SINGLE, "single")):
        out[f"round_{nm}"] = R.round(xs, p)

    # 2. the reference generator (build_convdiff3d, beta = 1, x = ones)
    for n in (3, 4, 8):
        A, b = R.convdiff(n)
        out[f"convdiff{n}_rp"], out[f"convdiff{n}_ci"], out[f"convdiff{n}_v"], out[f"convdiff{n}_b"] = A.rp, A.ci, A.v, b

    # 3. kernels on convdiff n = 5 (N = 125, not a power of two) and n = 8
    for n in (5, 8):
        A, _ = R.convdiff(n)
        x = rng.uniform(-1, 1, A.n)
        bb = rng.uniform(-3, 3, A.n)
        out[f"k{n}_x"], out[f"k{n}_b"] = x, bb
        for p, nm in ((HALF, "h"), (SINGLE, "s"), (DOUBLE, "d")):
            xr = R.round(x, p)
            out[f"k{n}_xr_{nm}"] = xr
            out[f"k{n}_matvec_{nm}"] = R.matvec(A, xr, p)
            out[f"k{n}_resid_{nm}"] = R.residual(A, xr, bb, p, DOUBLE)
            out[f"k{n}_dot_{nm}"] = np.array([R.dot(xr, R.round(bb, p), p)])
            out[f"k{n}_norm2_{nm}"] = np.array([R.norm2(R.round(bb, p), p)])
        H, S = R.regularize(A, 0.5)
        out[f"k{n}_H_rp"], out[f"k{n}_H_ci"], out[f"k{n}_H_v"], out[f"k{n}_S_v"] = H.rp, H.ci, H.v, S.v
        for p, nm in ((HALF, "h"), (SINGLE, "s"), (DOUBLE, "d")):
            rhs = R.round(rng.uniform(-1, 1, A.n), p)
            stop = R.norm2_64(rhs)
            out[f"k{n}_rhs_{nm}"] = rhs
            for meth, mn, M in ((CG, "cg", H), (GMRES, "gm", S)):
                x, it, st = R.krylov(M, rhs, meth, 1e-6, 60, 10, p, stop)
                out[f"k{n}_{mn}_{nm}_x"] = x
                out[f"k{n}_{mn}_{nm}_info"] = np.array([it, st])

    # 4. whole solves on seeded systems from the shared splitmix64 generator
    solves = [("s16", 16, SINGLE, 0.1, 0, 0.0, 1.0), ("h16", 16, HALF, 0.1, 0, 0.0, 1.0),
              ("d8", 8, DOUBLE, 0.5, 0, 0.0, 1.0), ("s8b", 8, SINGLE, 0.2, 1, -1.0, 1.0)]
    for tag, n, ur, alpha, seed, lo, hi in solves:
        A = o.convdiff(n)
        _, b = o.make_rhs(A, seed, lo, hi)
        cfg = Config.make(alpha=alpha, xi=1e-20, u_r=ur, method=CG, tol_epsilon=1e-12, max_inner_iters=50)
        x, rep, hist = R.solve(A, b, cfg)
        out[f"solve_{tag}_b"] = b
        out[f"solve_{tag}_x"] = x
        out[f"solve_{tag}_hist"] = hist
        out[f"solve_{tag}_info"] = np.array([rep.status, rep.outer_iters, rep.inner_iter_totals,
                                             rep.inner_stagnations], dtype=np.int64)
        out[f"solve_{tag}_cfg"] = np.array([n, ur, alpha, seed, lo, hi])

    # 6. LuDirect (BandLU, band_lu.cpp; the reference's default inner method):
    #    factor + solve of H and S of sections 3 (n = 5, 8), a pivoting case
    #    (strong convection, small alpha: S is far from diagonally dominant),
    #    the two exceptions, and whole solves with inner lu.
    lu_mats = {}
    for n in (5, 8):
        H = CSR(out[f"k{n}_H_rp"].size - 1, out[f"k{n}_H_rp"], out[f"k{n}_H_ci"], out[f"k{n}_H_v"])
        S = CSR(H.n, H.rp, H.ci, out[f"k{n}_S_v"])
        lu_mats[f"k{n}H"], lu_mats[f"k{n}S"] = H, S
    Ap = o.convdiff(6, r=0.45)
    Hp, Sp = R.regularize(Ap, 0.02)
    lu_mats["pivH"], lu_mats["pivS"] = Hp, Sp
    out["lu_piv_rp"], out["lu_piv_ci"], out["lu_piv_H"], out["lu_piv_S"] = Hp.rp, Hp.ci, Hp.v, Sp.v
    out["lu_sing_v"] = np.array([1e-6, 2.0, 3.0])           # diagonal: below binary16 min_normal
    out["lu_ovf_v"] = np.array([1.0, 60000.0, 0.5, -60000.0])  # U22 = -90000 overflows binary16
    lu_mats["sing"] = CSR(3, np.array([0, 1, 2, 3]), np.array([0, 1, 2]), out["lu_sing_v"])
    lu_mats["ovf"] = CSR(2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), out["lu_ovf_v"])
    for tag, M in lu_mats.items():
        for p, nm in ((HALF, "h"), (SINGLE, "s"), (DOUBLE, "d")):
            rhs = R.round(rng.uniform(-1, 1, M.n), p)
            x, st = R.lu_solve(M, rhs, p)
            out[f"lu_{tag}_{nm}_rhs"], out[f"lu_{tag}_{nm}_x"], out[f"lu_{tag}_{nm}_st"] = rhs, x, np.array([st])
    lu_solves = [("luh8", 8, HALF, 0.1), ("lus8", 8, SINGLE, 0.1), ("lud6", 6, DOUBLE, 0.5), ("luh12", 12, HALF, 0.3)]
    for tag, n, ur, alpha in lu_solves:
        A = o.convdiff(n)
        _, b = o.make_rhs(A, 0, 0.0, 1.0)
        cfg = Config.make(alpha=alpha, xi=1e-20 if ur != HALF else 1e-8, u_r=ur, method=LU)
        x, rep, hist = R.solve(A, b, cfg)
        out[f"solve_{tag}_b"], out[f"solve_{tag}_x"], out[f"solve_{tag}_hist"] = b, x, hist
        out[f"solve_{tag}_info"] = np.array([rep.status, rep.outer_iters, rep.inner_iter_totals,
                                             rep.inner_stagnations], dtype=np.int64)
        out[f"solve_{tag}_cfg"] = np.array([n, ur, alpha, 0, 0.0, 1.0])

    # 5. GPR fit/predict through the reference's gpr.cpp (Eigen restated in oracle/eigen_shim)
    sizes = np.array([8 ** 3, 12 ** 3, 16 ** 3, 24 ** 3, 32 ** 3, 48 ** 3, 64 ** 3], dtype=np.int64)
    alphas = 0.5 * sizes.astype(np.float64) ** (-1.0 / 3.0) * (1.0 + 0.05 * rng.standard_normal(len(sizes)))
    q = np.array([10 ** 3, 20 ** 3, 40 ** 3, 100 ** 3, 200 ** 3], dtype=np.int64)
    mean, sd, params = R.gpr(sizes, alphas, q)
    out["gpr_sizes"], out["gpr_alphas"], out["gpr_q"] = sizes, alphas, q
    out["gpr_mean"], out["gpr_sd"], out["gpr_params"] = mean, sd, params

    # 7. GPR training-set generation: alpha_bisection (gpr.cpp:15-50) on the
    #    convdiff family, each probe a uniform-precision solve
    bis = [("bs6", 6, SINGLE, 1e-2, 1e2, 17, dict(train_xi=1e-8, max_outer=1500)),          # test_gpr.cpp:53-63
           ("bd5", 5, DOUBLE, 1e-2, 1e2, 9, dict(train_xi=1e-8, max_outer=800)),
           ("bh4", 4, HALF, 1e-2, 1e2, 9, dict(train_xi=1e-3, max_outer=800)),
           ("bcg5", 5, SINGLE, 1e-2, 1e2, 9, dict(method=CG, tol_epsilon=1e-6, max_inner_iters=50, max_outer=800))]
    for tag, n, fmt, lo, hi, budget, kw in bis:
        a, it = R.alpha_bisection(n, fmt, lo, hi, budget, Dichotomy.make(**kw))
        out[f"bis_{tag}"] = np.array([n, fmt, lo, hi, budget, a, it], dtype=np.float64)
    for n in (4, 5, 6):  # generate_training_set({4,5,6}, single, budget 9), test_gpr.cpp:144-160
        a, it = R.alpha_bisection(n, SINGLE, 1e-2, 1e2, 9, Dichotomy.make(budget=9, train_xi=1e-8, max_outer=800))
        out[f"ts_{n}"] = np.array([n ** 3, a, it], dtype=np.float64)

    # 8. Sylvester GADI-AB (sylvester.cpp, problems.cpp:45-66): test_problems.cpp:152-160
    #    and acceptance criterion 7's table configuration (n = 64, half/double/double)
    syl = [("s16", 16, 0.1, dict(alpha=0.5, xi=1e-22, max_outer_iters=20000)),
           ("c7a", 64, 0.1, dict(alpha=0.02, xi=0.0, u_r=HALF, max_outer_iters=30000, stall_window=400,
                                 residual_scaling=0)),
           ("c7b", 64, 1.0, dict(alpha=10.0, xi=0.0, u_r=HALF, max_outer_iters=30000, stall_window=400,
                                 residual_scaling=0)),
           ("sgl", 24, 0.5, dict(alpha=0.3, xi=1e-12, u_r=SINGLE, u=SINGLE, u_f=SINGLE, max_outer_iters=5000))]
    for tag, n, r, kw in syl:
        X, rep, hist = R.sylvester_solve(n, r, Config.make(**kw))
        out[f"syl_{tag}_X"], out[f"syl_{tag}_hist"] = X, hist
        out[f"syl_{tag}_info"] = np.array([rep.status, rep.outer_iters, rep.inner_iter_totals, rep.inner_stagnations])

    path = os.path.join(HERE, "reference_vectors.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
