"""Summarise an ncu --metrics launch list CSV: last N launches, per kernel."""
import csv, sys
from collections import OrderedDict
path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
ik, im, iv, iid = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
ig, ib = hdr.index("Grid Size"), hdr.index("Block Size")
d = OrderedDict()
for r in rows[1:]:
    key = (int(r[iid]), r[ik].split("(")[0].replace("void ", "")[-30:], r[ig], r[ib])
    d.setdefault(key, {})[r[im].split(".")[0]] = r[iv]
for (i, k, g, b), m in list(d.items())[-n:]:
    print(f"{i:4d} {k:30s} grid{g:>14s} blk{b:>14s}", " ".join(f"{kk[-24:]}={vv}" for kk, vv in m.items()))
