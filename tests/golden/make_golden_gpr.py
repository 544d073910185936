"""Golden predictions for BASELINE configs[4] (tests/golden/gpr_c5.npz).

m = 4096 training pairs, log10 N ~ U[4,8], alpha = 0.5 N^(-1/3) (1 + 0.05 N(0,1))
(seed 3), fixed hyperparameters sigma_f^2 = var(y), l = 1, sigma_n^2 = 1e-4,
65,536 query sizes (bench.c5_data). The reference's fit (gpr.cpp:109-149)
cannot take a fixed length scale, so the values come from the oracle
restatement of try_fit / predict_alpha (oracle/gadi_oracle.c, pinned to the
reference's own fit on the grid-mode vectors in test_oracle_pin.py), evaluated
at 384 of the queries (one binary64 triangular solve each).

    python tests/golden/make_golden_gpr.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from bench import c5_data  # noqa: E402
from oracle import Oracle  # noqa: E402


def main():
    sizes, alphas, q, fixed = c5_data()
    idx = np.unique(np.concatenate([np.arange(0, len(q), 172), np.argsort(q)[[0, 1, -2, -1]]]))
    mean, sd, params = Oracle().gpr(sizes, alphas, q[idx], fixed=fixed)
    path = os.path.join(HERE, "gpr_c5.npz")
    np.savez_compressed(path, idx=idx, mean=mean, sd=sd, params=params, fixed=np.array(fixed),
                        sizes_sum=np.array([sizes.sum(), alphas.sum(), q.sum()]))
    print("wrote", path, len(idx), "queries; sd range", sd.min(), sd.max(), "params", params)


if __name__ == "__main__":
    main()
