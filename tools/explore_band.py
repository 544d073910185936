"""C4 exploration (not a test): python tools/explore_band.py N ur accum alpha[,..] max_inner [max_outer]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_04229_b200 as g
N, ur, acc = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
alphas = [float(a) for a in sys.argv[4].split(",")]
mi = int(sys.argv[5]); mo = int(sys.argv[6]) if len(sys.argv) > 6 else 2000
t = time.time()
B = g.build_band_csr(N)
s = g.CudaGadiSystem(B)
torch.cuda.synchronize()
print(f"create+split N={N}: {time.time()-t:.2f}s", flush=True)
xt = torch.empty(N, dtype=torch.float64, device="cuda"); b = torch.empty_like(xt); x = torch.empty_like(xt)
s.make_rhs(2, -1.0, 1.0, xt.data_ptr(), b.data_ptr())
for a in alphas:
    cfg = g.GadiConfig(alpha=a, xi=1e-20, u_r=g.Precision(ur), accum=g.Accum(acc),
                       inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, mi, 30), max_outer_iters=mo, stall_window=400)
    t = time.time(); rep = s.solve_device(b.data_ptr(), x.data_ptr(), cfg); dt = time.time() - t
    err = (torch.linalg.norm(x - xt) / torch.linalg.norm(xt)).item()
    print(f"alpha={a} mi={mi}: {rep.status.name} outer={rep.outer_iters} cg={rep.h_iters} gm={rep.s_iters} "
          f"rres={rep.final_rres:.3e} err={err:.2e} dev={rep.solve_ms/1e3:.2f}s h={rep.h_ms:.0f} s={rep.s_ms:.0f} "
          f"o={rep.outer_ms:.0f} (first solve includes prepare)", flush=True)
