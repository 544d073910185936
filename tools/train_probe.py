"""Time generate_training_set on the device for a few worker counts (and
optionally one precision / size list) -- debugging aid for gadi_train.cu."""
import os
import sys
import time

sys.path.insert(0, ".")
import paper_2501_04229_b200 as g  # noqa: E402

fmt = g.Precision(int(sys.argv[1])) if len(sys.argv) > 1 else g.Precision.Single
sizes = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [4, 6, 8, 10, 12, 16]
st = g.DichotomySettings()
for n in sizes:
    t = time.time()
    try:
        a = g.alpha_bisection(n, fmt, st.alpha_lo, st.alpha_hi, st.budget, st)
    except Exception as e:  # noqa: BLE001
        a = repr(e)
    print(fmt.name, n, a, f"{time.time() - t:.2f} s", os.environ.get("GADI_TRAIN_WORKERS"), flush=True)
