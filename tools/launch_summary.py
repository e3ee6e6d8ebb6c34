"""Aggregate an ncu launch list (gpu__time_duration.sum per launch) by kernel:
count, total and mean device time, share.  Usage: launch_summary.py CSV [first_id last_id]"""
import csv, sys
from collections import defaultdict
path = sys.argv[1]
lo = int(sys.argv[2]) if len(sys.argv) > 2 else -1
hi = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 60
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
ik, im, iv, iid = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum" or not (lo <= int(r[iid]) <= hi):
        continue
    name = r[ik].split("(")[0].replace("void ", "").strip()
    agg[name][0] += 1
    agg[name][1] += float(r[iv]) / 1e3  # ns -> us
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':44s} {'launches':>8s} {'total_us':>12s} {'mean_us':>10s} {'share':>7s}")
for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name[:44]:44s} {c:8d} {t:12.1f} {t / c:10.2f} {100 * t / tot:6.1f}%")
print(f"{'total':44s} {sum(v[0] for v in agg.values()):8d} {tot:12.1f}")
