"""Incremental cell sums A/B: the same design with VQB_DELTA=0 (every pass sums all rows)
and the default, on one session: wall time, per-level time per pass, and bit equality of
the codebook, the history and the per-row distances.  Usage: delta_ab.py cfg2 [frac ...]"""
import os, sys, time
from collections import defaultdict
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_4711_b200 as vq
from paper_0910_4711_b200 import synthetic
from paper_0910_4711_b200.core import _Session

which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
fracs = sys.argv[2:] or ["0.3"]
spec = synthetic.WORKLOADS[which]
s = _Session(synthetic.make_training(which), None)
conf = vq.LbgConfig(target_size=spec.target_size, epsilon=spec.epsilon, delta=spec.delta)


def run(env):
    os.environ.update(env)
    best = None
    for _ in range(2):
        t0 = time.perf_counter()
        out = s.train(conf)
        dt = time.perf_counter() - t0
        if best is None or dt < best[0]:
            best = (dt, out)
    return best


def levels(hist):
    prev, agg, cnt = 0.0, defaultdict(float), defaultdict(int)
    for h in hist:
        agg[h.codebook_size] += h.seconds - prev
        cnt[h.codebook_size] += 1
        prev = h.seconds
    return {k: (cnt[k], 1e6 * agg[k] / cnt[k]) for k in sorted(agg)}


t_ref, ref = run({"VQB_DELTA": "0"})
print(which, "full sums every pass:", round(t_ref * 1e3, 2), "ms")
lv0 = levels(ref[1])
for f in fracs:
    t, out = run({"VQB_DELTA": "1", "VQB_DELTA_FRAC": f})
    same_cb = np.array_equal(np.asarray(ref[0]), np.asarray(out[0]))
    same_hist = [(h.codebook_size, h.iteration, h.td, h.empty_cells) for h in ref[1]] == \
                [(h.codebook_size, h.iteration, h.td, h.empty_cells) for h in out[1]]
    same_d = np.array_equal(np.asarray(ref[4]), np.asarray(out[4])) if ref[4] is not None else None
    print(which, f"incremental (frac {f}):", round(t * 1e3, 2), "ms; codebook equal", same_cb,
          "history equal", same_hist, "distances equal", same_d, "total equal", ref[3] == out[3])
    lv1 = levels(out[1])
    for k in lv0:
        print(f"  K={k:5d} passes={lv0[k][0]:3d} us/pass full={lv0[k][1]:8.1f} incremental={lv1[k][1]:8.1f}")
