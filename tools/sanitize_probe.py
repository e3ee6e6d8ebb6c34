"""Small-size exercise of every device path for compute-sanitizer
(racecheck / synccheck / memcheck, one tool per gpurun call): assign_tc<16>
(resident codebook) and <64>, the streaming ring (K = 4096), assign_fast,
the shortlist / exact re-rank, the limb-RED and warp-table cell sums, the
reference-order path (float64 rows), a full design, encode."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_0910_4711_b200 as vq  # noqa: E402
from paper_0910_4711_b200 import synthetic  # noqa: E402

rng = np.random.default_rng(1)
x16 = synthetic.make_training("cfg2", n=8192)
ts = vq.TrainingSet(x16)
for k in (16, 256, 4096):  # assign_fast / assign_tc<16> resident / streaming ring
    t, _ = vq.assign_cells(ts, vq.Codebook(rng.uniform(0, 255, (k, 16))))
    vq.update_codebook(ts, t, vq.Codebook(rng.uniform(0, 255, (k, 16))))  # RED / warp-table sums
x64 = synthetic.make_training("cfg3", n=4096)[:4096]
t, _ = vq.assign_cells(x64, vq.Codebook(x64[:512].astype(np.float64) + 0.5))  # assign_tc<64>
cb, st = vq.lbg_train(ts, vq.LbgConfig(target_size=64, epsilon=1e-3))
xd = rng.normal(0, 1, (3000, 5))  # float64 rows: exact scan + reference-order sums
cbd, _ = vq.lbg_train(vq.TrainingSet(xd), vq.LbgConfig(target_size=8))
s = vq.encode(x16, cb)
print("sanitize probe ok", len(st.history), int(s.indices.sum()))
