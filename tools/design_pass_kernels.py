"""Per-pass kernel breakdown of one design from an ncu launch list
(tools/profile_design.py under ncu --metrics gpu__time_duration.sum): for every
`every`-th pass, each kernel's device time (us).  Usage: design_pass_kernels.py CSV [every]"""
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
every = int(sys.argv[2]) if len(sys.argv) > 2 else 10
rows = list(csv.reader(lines))
hdr = rows[0]
ik, im, iv = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value"))
seq = [(r[ik].split("(")[0].replace("void ", "").replace("vqb::", ""), float(r[iv]) / 1e3)
       for r in rows[1:] if r[im] == "gpu__time_duration.sum"]
passes, cur = [], []
for n, t in seq:
    cur.append((n, t))
    if n == "apply_kernel":
        passes.append(cur)
        cur = []
for i, p in enumerate(passes):
    if i % every:
        continue
    d = {}
    for n, t in p:
        d[n] = d.get(n, 0) + t
    tot = sum(d.values())
    print(i, "tot", round(tot, 1), " ".join(f"{k.replace('_kernel', '')}={v:.1f}" for k, v in sorted(d.items(), key=lambda kv: -kv[1])))
