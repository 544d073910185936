"""Convergence exploration at BASELINE sizes on the GPU (not a test).
usage: python tools/explore_alpha.py n beta ur accum alpha[,alpha...] max_outer max_inner [omega]"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_04229_b200 as g

n, beta = int(sys.argv[1]), float(sys.argv[2])
ur, acc = int(sys.argv[3]), int(sys.argv[4])
alphas = [float(a) for a in sys.argv[5].split(",")]
max_outer, max_inner = int(sys.argv[6]), int(sys.argv[7])
omega = float(sys.argv[8]) if len(sys.argv) > 8 else 1.0
S = g.build_convdiff3d(n, beta=beta)
sysx = g.CudaGadiSystem(S)
N = S.n_rows
xt = torch.empty(N, dtype=torch.float64, device="cuda")
b = torch.empty_like(xt)
x = torch.empty_like(xt)
sysx.make_rhs(1, -1.0, 1.0, xt.data_ptr(), b.data_ptr())
torch.cuda.synchronize()
for a in alphas:
    cfg = g.GadiConfig(alpha=a, omega=omega, xi=1e-20, u_r=g.Precision(ur), accum=g.Accum(acc),
                       inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, max_inner, 30),
                       max_outer_iters=max_outer, stall_window=400)
    t = time.time()
    rep = sysx.solve_device(b.data_ptr(), x.data_ptr(), cfg)
    dt = time.time() - t
    h = rep.rel_residual_history
    err = (torch.linalg.norm(x - xt) / torch.linalg.norm(xt)).item()
    idx = [i for i in (1, 10, 50, 100, 200, 400, 800, 1600, 3200, 6400) if i < len(h)] + [len(h) - 1]
    print(f"n={n} beta={beta} ur={ur} acc={acc} omega={omega} alpha={a}: status={rep.status.name} outer={rep.outer_iters} "
          f"inner={rep.inner_iter_totals} (H {rep.h_iters}, S {rep.s_iters}) rres={rep.final_rres:.3e} "
          f"err={err:.2e} wall={dt:.2f}s dev={rep.solve_ms/1e3:.2f}s h_ms={rep.h_ms:.0f} s_ms={rep.s_ms:.0f}", flush=True)
    print("   hist:", " ".join(f"{i}:{h[i]:.2e}" for i in idx), flush=True)
