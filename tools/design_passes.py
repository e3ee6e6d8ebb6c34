"""Per-pass device times of one design from an ncu launch list
(tools/profile_design.py under ncu --metrics gpu__time_duration.sum).
Usage: design_passes.py CSV [every]"""
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
every = int(sys.argv[2]) if len(sys.argv) > 2 else 6
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
short = {"assign_tc_kernel<16, 0>": "tc", "assign_tc_kernel<16, 1>": "tcsl", "sums_kernel<float, 16>": "sums",
         "assign_fast_kernel<16, 1>": "fast"}
for i, p in enumerate(passes):
    if i % every:
        continue
    d = {}
    for n, t in p:
        k = short.get(n, None)
        if k:
            d[k] = d.get(k, 0) + t
    print(i, {k: round(v, 1) for k, v in d.items()}, "tot", round(sum(t for _, t in p), 1))
print("design total us", round(sum(t for _, t in seq), 1))
