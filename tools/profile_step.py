"""A short C3/C2 solve for profiling (ncu launch lists): W warm-up outer steps
then `--outer` more, max_outer capped (not a benchmark)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_04229_b200 as g
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_cfg import WORKLOADS  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3")
ap.add_argument("--outer", type=int, default=2)
ap.add_argument("--repeat", type=int, default=1)
a = ap.parse_args()
wl = WORKLOADS[a.workload]
if wl.get("kind") == "band":
    S = g.build_band_csr(wl["N"], wl["k_off"], wl["band"], wl["mseed"])
else:
    S = g.build_convdiff3d(wl["n"], beta=wl["beta"])
sysx = g.CudaGadiSystem(S)
xt = torch.empty(S.n_rows, dtype=torch.float64, device="cuda")
b = torch.empty_like(xt); x = torch.empty_like(xt)
sysx.make_rhs(wl["seed"], wl["lo"], wl["hi"], xt.data_ptr(), b.data_ptr())
cfg = g.GadiConfig(alpha=wl["alpha"], omega=wl.get("omega", 1.0), xi=1e-20, u_r=g.Precision(wl["u_r"]),
                   accum=g.Accum(wl["accum"]),
                   inner=g.InnerSolverSpec(g.InnerMethod.Cg, wl["eps"], wl["max_inner"], wl["restart"]),
                   max_outer_iters=a.outer)
for _ in range(a.repeat):
    rep = sysx.solve_device(b.data_ptr(), x.data_ptr(), cfg)
    print(f"outer={rep.outer_iters} cg={rep.h_iters} gmres={rep.s_iters} solve_ms={rep.solve_ms:.1f} "
      f"h_ms={rep.h_ms:.1f} s_ms={rep.s_ms:.1f} outer_ms={rep.outer_ms:.1f} launches={rep.launches}")
