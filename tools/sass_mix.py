"""Opcode mix (warp-level instructions executed) from an `ncu --page source --csv` export."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
for hi, r in enumerate(rows):
    if 'Source' in r and 'Address' in r:
        break
h = rows[hi]; data = rows[hi + 1:]
iS, iE = h.index('Source'), h.index('Instructions Executed')
iW = h.index('Warp Stall Sampling (All Samples)')
mix = collections.Counter(); st = collections.Counter()
for d in data:
    try:
        n = float(d[iE] or 0)
    except ValueError:
        continue
    src = d[iS].strip()
    if src.startswith('@'):
        src = src.split(None, 1)[1] if ' ' in src else src
    op = src.split(' ')[0]
    mix[op] += n
    try:
        st[op] += float(d[iW] or 0)
    except ValueError:
        pass
tot = sum(mix.values()); ts = sum(st.values()) or 1
print(f"total warp instructions {tot:.4g}")
for op, n in mix.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{op:28s} {n:12.4g} {n / tot:6.1%}  stall-samples {st[op] / ts:6.1%}")
