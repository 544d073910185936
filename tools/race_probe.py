"""Small solves for compute-sanitizer --tool racecheck / synccheck: the
pipelined band-LU sweeps (k_lu_pipe: (value | epoch) words polled across
CTAs), the ticketed last-block reductions (grid_finish) of the Krylov passes,
the st25 TMA rings, and a 2-rank local sharded solve."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2501_04229_b200 as g

rng = np.random.default_rng(0)
n = 12
S = g.build_convdiff3d(n)
b = rng.uniform(-1, 1, n ** 3)
r = g.gadi_ir_solve(S, b, g.hss_split(S), g.GadiConfig(alpha=0.3, xi=1e-8, u_r=g.Precision.Half, max_outer_iters=12))
print("lu half", r.report.status, r.report.outer_iters)
r = g.gadi_ir_solve(S, b, g.hss_split(S), g.GadiConfig(alpha=0.3, xi=1e-12, u_r=g.Precision.Single, max_outer_iters=6))
print("lu single", r.report.status, r.report.outer_iters)
n = 16
S = g.build_convdiff3d(n)
b = rng.uniform(-1, 1, n ** 3)
for ur, acc in ((g.Precision.Single, g.Accum.Native), (g.Precision.Half, g.Accum.Fp32), (g.Precision.Double, g.Accum.Native)):
    cfg = g.GadiConfig(alpha=0.2, xi=1e-20, u_r=ur, accum=acc, max_outer_iters=4,
                       inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 6, 4))
    r = g.gadi_ir_solve(S, b, g.hss_split(S), cfg)
    print("krylov", ur, r.report.status, r.report.outer_iters, r.report.inner_iter_totals)
B = g.build_band_csr(2048, 8, 64, 2)
bb = rng.uniform(-1, 1, 2048)
r = g.gadi_ir_solve(B, bb, g.hss_split(B), g.GadiConfig(alpha=2.0, xi=1e-20, u_r=g.Precision.Half, accum=g.Accum.Fp32,
                    max_outer_iters=3, inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 5, 4)))
print("band", r.report.status, r.report.outer_iters)
print("done")
