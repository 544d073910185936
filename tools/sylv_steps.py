import sys; sys.path.insert(0, ".")
import paper_2501_04229_b200 as g
res = g.gadi_ab_solve(g.build_sylvester(256, 0.1), g.GadiConfig(u_r=g.Precision.Half, residual_scaling=False, alpha=0.02, xi=0.0, max_outer_iters=3))
print(res.report.solve_ms, res.report.outer_iters)
