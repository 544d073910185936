"""C5-sized GPR fit + predict once (for ncu captures of the dense kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_04229_b200 as g
from bench import c5_data
sizes, alphas, q, fixed = c5_data()
m = g.gpr_fit(sizes, alphas, fixed=fixed)
mean, sd = m.predict(q)
print(m.timings(), float(sd.max()))
