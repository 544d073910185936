"""Sharded-vs-single diagnostic (not a test): python tools/dbg_shard.py n world ur accum max_outer"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_04229_b200 as g
n, world, ur, acc, mo = (int(a) for a in sys.argv[1:6])
S = g.build_convdiff3d(n, r=0.3)
N = S.n_rows
full = g.CudaGadiSystem(S)
xt = torch.empty(N, dtype=torch.float64, device="cuda"); b = torch.empty_like(xt)
full.make_rhs(1, -1.0, 1.0, xt.data_ptr(), b.data_ptr())
for mi, meth in ((5, g.InnerMethod.Cg),):
    cfg = g.GadiConfig(alpha=0.2, xi=1e-20, u_r=g.Precision(ur), accum=g.Accum(acc), stall_window=400,
                       inner=g.InnerSolverSpec(meth, 1e-12, mi, 30), max_outer_iters=mo)
    x1 = torch.empty_like(xt); r1 = full.solve_device(b.data_ptr(), x1.data_ptr(), cfg)
    grp = g.ShardGroup.local(world); sh = [g.ShardSystem(S, grp, r) for r in range(world)]
    nl = sh[0].n; xs = torch.empty_like(xt)
    reps = g.solve_group(sh, cfg, [b.data_ptr() + r * nl * 8 for r in range(world)], [xs.data_ptr() + r * nl * 8 for r in range(world)])
    torch.cuda.synchronize()
    a, c = x1.cpu().numpy(), xs.cpu().numpy()
    d = np.nonzero(a.view(np.int64) != c.view(np.int64))[0]
    print("outer", r1.outer_iters, reps[0].outer_iters, "inner", r1.inner_iter_totals, reps[0].inner_iter_totals,
          "ndiff", len(d), "first planes", sorted(set((d // (n * n)).tolist()))[:20])
    h1, h2 = r1.rel_residual_history, reps[0].rel_residual_history
    k = np.nonzero(h1.view(np.int64) != h2.view(np.int64))[0]
    print("hist first diff at", k[:5], h1[k[:3]] if len(k) else None, h2[k[:3]] if len(k) else None)
