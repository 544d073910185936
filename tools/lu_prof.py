"""One LuDirect prepare + one H solve at n = 32 in binary16 (for ncu)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2501_04229_b200 as g  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
ur = g.Precision(int(sys.argv[2])) if len(sys.argv) > 2 else g.Precision.Half
S = g.build_convdiff3d(n)
sysx = g.CudaGadiSystem(S)
sysx.prepare(0.1, 1.0, ur, g.InnerSolverSpec(g.InnerMethod.LuDirect, 1e-2, 1000, 30))
rhs = np.random.default_rng(1).uniform(-1, 1, n ** 3).astype(np.float16).astype(np.float64)
sysx.solve_H(rhs)
