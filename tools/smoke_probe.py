import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, paper_2501_04229_b200 as g
from oracle import Oracle
orc=Oracle(); n=16
S=g.build_convdiff3d(n); A=orc.convdiff(n,S.t1,S.t2,S.t3); _,b=orc.make_rhs(A,0,0.0,1.0)
cfg=g.GadiConfig(alpha=0.1,xi=1e-20,u_r=g.Precision.Single,inner=g.InnerSolverSpec(g.InnerMethod.Cg,1e-12,50,30))
for _ in range(3):
    res=g.gadi_ir_solve(S,b,g.hss_split(S),cfg,device=0); r=res.report
    print(r.outer_iters, r.h_iters, r.s_iters, r.launches, round(r.solve_ms,1), round(r.h_ms,1), round(r.s_ms,1), round(r.outer_ms,1))
