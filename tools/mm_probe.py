"""Time MatrixMarket ingest: gadi_mm_read (host parse + device from_triplets
assembly) against the reference's read_matrix_market_file (oracle/_ref/ref_mm,
one host core) on a synthetic 2^20-row, ~10M-entry general file with
duplicates; checks the two CSRs are identical."""
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2501_04229_b200 as g  # noqa: E402

n, m = 1 << 20, 10_000_000
rng = np.random.default_rng(7)
i = rng.integers(1, n + 1, m)
j = np.clip(i + rng.integers(-64, 65, m), 1, n)
v = rng.integers(-512, 513, m) / 64.0  # dyadic: duplicate sums are exact in any order
d = tempfile.mkdtemp()
path = os.path.join(d, "big.mtx")
t = time.perf_counter()
with open(path, "w") as f:
    f.write(f"%%MatrixMarket matrix coordinate real general\n{n} {n} {m}\n")
    np.savetxt(f, np.column_stack([i, j, v]), fmt=["%d", "%d", "%.17g"])
print(f"wrote {os.path.getsize(path) / 1e6:.0f} MB in {time.perf_counter() - t:.1f} s", flush=True)
g.read_matrix_market_file(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "mm", "general.mtx"))
t = time.perf_counter()
A = g.read_matrix_market_file(path)
td = time.perf_counter() - t
print(f"gadi_mm_read: {td:.2f} s, nnz {A.nnz()}", flush=True)
ref = os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "ref_mm")
if os.path.exists(ref):
    out = os.path.join(d, "ref.bin")
    t = time.perf_counter()
    subprocess.run([ref, path, out], check=True)
    tr = time.perf_counter() - t
    raw = np.fromfile(out, np.int64)
    nnz = int(raw[0])
    rp = raw[3:3 + n + 1]
    ci = raw[4 + n:4 + n + nnz]
    vv = raw[4 + n + nnz:4 + n + 2 * nnz]
    same = np.array_equal(rp, A.row_ptr) and np.array_equal(ci, A.col_idx) and np.array_equal(vv, A.values.view(np.int64))
    print(f"reference read_matrix_market_file: {tr:.2f} s (incl. binary dump), identical CSR: {same}")
