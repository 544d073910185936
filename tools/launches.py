"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = []
for r in rows:
    if r and r[0] == 'ID':
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    k = d['Kernel Name'].split('(')[0][:70]
    agg.setdefault(k, collections.defaultdict(list))[d['Metric Name']].append(float(d['Metric Value'].replace(',', '')))
tot = sum(sum(v['gpu__time_duration.sum']) for v in agg.values())
print(f"{'kernel':70s} {'n':>4s} {'avg_us':>9s} {'share':>6s} {'rdMB':>8s} {'wrMB':>8s} {'GB/s':>6s}")
for k, v in agg.items():
    t = v['gpu__time_duration.sum']; rd = v.get('dram__bytes_read.sum', [0]); wr = v.get('dram__bytes_write.sum', [0])
    print(f"{k:70s} {len(t):4d} {sum(t)/len(t)/1e3:9.1f} {sum(t)/tot:6.1%} {sum(rd)/len(rd)/1e6:8.1f} {sum(wr)/len(wr)/1e6:8.1f} {(sum(rd)+sum(wr))/sum(t):6.0f}")
