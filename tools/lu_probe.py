"""Time the device LuDirect path on C1 (n = 32 convdiff, BASELINE configs[0]):
prepare (two band factorizations) and whole GADI-IR solves in each u_r."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2501_04229_b200 as g  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
S = g.build_convdiff3d(n)
LU = g.InnerSolverSpec(g.InnerMethod.LuDirect, 1e-2, 1000, 30)
sysx = g.CudaGadiSystem(S)
N = n ** 3
b = np.random.default_rng(0).uniform(0, 1, N)
for ur in (g.Precision.Half, g.Precision.Single, g.Precision.Double):
    t = time.perf_counter()
    sysx.prepare(0.1, 1.0, ur, LU)
    tp = time.perf_counter() - t
    rhs = np.random.default_rng(1).uniform(-1, 1, N).astype(np.float16 if ur == 0 else np.float32).astype(np.float64)
    t = time.perf_counter()
    for _ in range(5):
        sysx.solve_H(rhs)
    ts = (time.perf_counter() - t) / 5
    cfg = g.GadiConfig(alpha=0.1, xi=1e-20 if ur else 1e-8, u_r=ur, inner=LU)
    t = time.perf_counter()
    res = g.gadi_ir_solve(S, b, g.hss_split(S), cfg)
    tt = time.perf_counter() - t
    r = res.report
    print(f"n={n} u_r={ur.name}: prepare {tp*1e3:.1f} ms, one inner solve (host copies incl.) {ts*1e3:.2f} ms; "
          f"solve {r.status.name} outer={r.outer_iters} rres={r.final_rres:.2e} device {r.solve_ms:.1f} ms "
          f"(H {r.h_ms:.1f}, S {r.s_ms:.1f}) wall {tt*1e3:.0f} ms launches={r.launches}", flush=True)
