"""CPU restatement of the reference's MatrixMarket reader/writer
(matrix_market.cpp:22-86) and SparseMatrix::from_triplets (sparse.cpp:36-58).
TEST INFRASTRUCTURE ONLY (pure Python; small files). Duplicates are summed in
file order (a stable sort); the reference's std::sort leaves that order
unspecified, so the fixtures use duplicates with exact sums."""
import numpy as np

IO_ERROR, CONTRACT = -12, -1


def read(path):
    """(n_rows, n_cols, rp, ci, v) or an error code (IoError -12, ContractViolation -1)."""
    with open(path) as f:
        text = f.read().split("\n")
    if not text or (len(text) == 1 and text[0] == ""):
        return IO_ERROR
    hdr = text[0].split()
    hdr += [""] * (5 - len(hdr))
    banner, obj, fmt, field, sym = hdr[:5]
    if banner != "%%MatrixMarket" or obj.lower() != "matrix":
        return IO_ERROR
    if fmt.lower() != "coordinate":
        return IO_ERROR
    field, sym = field.lower(), sym.lower()
    if field not in ("real", "integer"):
        return IO_ERROR
    if sym not in ("general", "symmetric", "skew-symmetric"):
        return IO_ERROR
    k = 1
    while k < len(text) and (text[k] == "" or text[k][0] == "%"):
        k += 1
    try:
        rows, cols, entries = (int(t) for t in text[k].split()[:3])
    except (ValueError, IndexError):
        return IO_ERROR
    toks = " ".join(text[k + 1:]).split()
    if len(toks) < 3 * entries:
        return IO_ERROR
    t = []
    for e in range(entries):
        i, j, v = int(toks[3 * e]) - 1, int(toks[3 * e + 1]) - 1, float(toks[3 * e + 2])
        t.append((i, j, v))
        if i != j and sym == "symmetric":
            t.append((j, i, v))
        if i != j and sym == "skew-symmetric":
            t.append((j, i, -v))
    t.sort(key=lambda e: (e[0], e[1]))  # stable
    rp = np.zeros(rows + 1, np.int64)
    ci, vals = [], []
    q = 0
    while q < len(t):
        i, j, s = t[q]
        q += 1
        while q < len(t) and t[q][0] == i and t[q][1] == j:
            s += t[q][2]
            q += 1
        if i < 0 or i >= rows or j < 0 or j >= cols:
            return CONTRACT
        ci.append(j)
        vals.append(s)
        rp[i + 1] += 1
    return rows, cols, np.cumsum(rp), np.array(ci, np.int64), np.array(vals, np.float64)


def write_text(n_rows, n_cols, rp, ci, v):
    """write_matrix_market (matrix_market.cpp:64-79)."""
    sym = n_rows == n_cols
    if sym:
        d = {}
        for i in range(n_rows):
            for k in range(rp[i], rp[i + 1]):
                d[(i, int(ci[k]))] = v[k]
        sym = all(d.get((j, i)) == x for (i, j), x in d.items())
    out = [f"%%MatrixMarket matrix coordinate real {'symmetric' if sym else 'general'}"]
    body = []
    for i in range(n_rows):
        for k in range(rp[i], rp[i + 1]):
            j = int(ci[k])
            if sym and j > i:
                continue
            body.append(f"{i + 1} {j + 1} {float(v[k]):.17g}")
    out.append(f"{n_rows} {n_cols} {len(body)}")
    return "\n".join(out + body) + "\n"
