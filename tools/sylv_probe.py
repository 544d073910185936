"""Time Sylvester GADI-AB (acceptance criterion 7 cells, n = 64, and larger n) on
the device next to the reference's own gadi_ab_solve (oracle/_ref, one core)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2501_04229_b200 as g  # noqa: E402
from oracle import DOUBLE, HALF, Config, Reference  # noqa: E402

R = Reference() if Reference.available() else None
for n, r, a in ((64, 0.1, 0.02), (64, 1.0, 10.0), (128, 0.1, 0.02), (256, 0.1, 0.02)):
    kw = dict(alpha=a, xi=0.0, max_outer_iters=30000, stall_window=400)
    t = time.perf_counter()
    res = g.gadi_ab_solve(g.build_sylvester(n, r), g.GadiConfig(u_r=g.Precision.Half, residual_scaling=False, **kw))
    td = time.perf_counter() - t
    line = (f"n={n} r={r} alpha={a}: device {res.report.status.name} outer={res.report.outer_iters} "
            f"rres={res.report.final_rres:.3e} {td:.2f} s (device {res.report.solve_ms / 1e3:.2f} s)")
    if R is not None and n <= 128:
        t = time.perf_counter()
        _, rep, _ = R.sylvester_solve(n, r, Config.make(u_r=HALF, u=DOUBLE, u_f=DOUBLE, residual_scaling=0, **kw))
        line += f"; reference outer={rep.outer_iters} {time.perf_counter() - t:.2f} s"
    print(line, flush=True)
