"""Write the MatrixMarket fixtures in tests/golden/mm/ and the reference's
read_matrix_market_file output for each (tests/golden/mm_reference.npz).

The files are synthetic (seeded); duplicate entries carry dyadic values so
their sums are exact in any order (the reference's std::sort leaves the order
of equal keys unspecified).

    make -f oracle/Makefile.ref all mm && python tests/golden/make_mm.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import subprocess  # noqa: E402
import tempfile  # noqa: E402

REF_MM = os.path.join(os.path.dirname(os.path.dirname(HERE)), "oracle", "_ref", "ref_mm")


def ref_read(path):
    """The reference's read_matrix_market_file through oracle/_ref/ref_mm (a
    subprocess: the reference library's static libstdc++ cannot share a
    process with numpy's)."""
    with tempfile.NamedTemporaryFile(suffix=".bin") as t:
        subprocess.run([REF_MM, path, t.name], check=True)
        raw = np.fromfile(t.name, np.int64)
    nnz = int(raw[0])
    if nnz < 0:
        return nnz
    nr, nc = int(raw[1]), int(raw[2])
    rp = raw[3:3 + nr + 1]
    ci = raw[4 + nr:4 + nr + nnz]
    v = raw[4 + nr + nnz:4 + nr + 2 * nnz].view(np.float64)
    return nr, nc, rp.copy(), ci.copy(), v.copy()

MM = os.path.join(HERE, "mm")


def write(name, text):
    with open(os.path.join(MM, name), "w") as f:
        f.write(text)


def main():
    os.makedirs(MM, exist_ok=True)
    rng = np.random.default_rng(42)
    write("general.mtx", "%%MatrixMarket matrix coordinate real general\n% a comment\n%\n\n"
          "4 5 8\n3 2 -1.5\n1 1 2.0\n4 5 1e-3\n1 1 0.25\n2 4 7\n1 3 -0.5\n4 1 3.25e2\n3 2 0.125\n")
    write("symmetric.mtx", "%%MatrixMarket matrix coordinate real symmetric\n3 3 5\n1 1 4\n2 1 -1\n"
          "3 3 4\n3 2 -1.25\n2 2 4\n")
    write("skew.mtx", "%%MatrixMarket MATRIX Coordinate Real Skew-Symmetric\n3 3 2\n2 1 0.5\n3 1 -2\n")
    write("integer.mtx", "%%MatrixMarket matrix coordinate integer general\n2 2 3\n1 2 3\n2 1 -4\n2 2 1\n")
    # tokens the parallel parser hands back to the stream loop: '+' signs, entries across lines
    write("stream_tokens.mtx", "%%MatrixMarket matrix coordinate real general\n3 3 4\n+1 1 +2.5\n2\n2 -1e+1 3 3\n"
          "0.5 1 3 +4.\n")
    write("empty.mtx", "%%MatrixMarket matrix coordinate real general\n3 3 0\n")
    # a larger random file: 2000 x 2000, 30000 entries, ~10% duplicates, dyadic values
    n, m = 2000, 30000
    i = rng.integers(1, n + 1, m)
    j = rng.integers(1, n + 1, m)
    dup = rng.random(m) < 0.1
    i[dup] = np.roll(i, 1)[dup]
    j[dup] = np.roll(j, 1)[dup]
    v = rng.integers(-64, 65, m) / 8.0
    lines = "".join(f"{a} {b} {float(c)!r}\n" for a, b, c in zip(i, j, v))
    write("random.mtx", f"%%MatrixMarket matrix coordinate real general\n{n} {n} {m}\n" + lines)
    # error cases (IoError / ContractViolation)
    write("bad_banner.mtx", "%%MatrixMarket vector coordinate real general\n2 2 1\n1 1 1\n")
    write("bad_format.mtx", "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n")
    write("bad_field.mtx", "%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 1 0\n")
    write("bad_sym.mtx", "%%MatrixMarket matrix coordinate real hermitian\n2 2 1\n1 1 1\n")
    write("truncated.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 2\n")
    write("out_of_range.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n3 1 2\n")
    out = {}
    for name in sorted(os.listdir(MM)):
        res = ref_read(os.path.join(MM, name))
        key = name[:-4]
        if isinstance(res, int):
            out[f"{key}_err"] = np.array([res])
        else:
            nr, nc, rp, ci, v = res
            out[f"{key}_shape"] = np.array([nr, nc])
            out[f"{key}_rp"], out[f"{key}_ci"], out[f"{key}_v"] = rp, ci, v
    np.savez_compressed(os.path.join(HERE, "mm_reference.npz"), **out)
    print({k: v.tolist() for k, v in out.items() if k.endswith("_err")})


if __name__ == "__main__":
    main()
