"""Per-level device time per pass of one design (history timestamps, %globaltimer)."""
import os, sys
from collections import defaultdict
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_4711_b200 as vq
from paper_0910_4711_b200 import synthetic
from paper_0910_4711_b200.core import _Session
which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
spec = synthetic.WORKLOADS[which]
s = _Session(synthetic.make_training(which), None)
conf = vq.LbgConfig(target_size=spec.target_size, epsilon=spec.epsilon, delta=spec.delta)
for _ in range(2):
    cb, hist, warns, total, d, summ = s.train(conf)
prev, agg, cnt = 0.0, defaultdict(float), defaultdict(int)
for h in hist:
    agg[h.codebook_size] += h.seconds - prev
    cnt[h.codebook_size] += 1
    prev = h.seconds
print(which, "total", round(prev * 1e3, 2), "ms")
for k in sorted(agg):
    print(f"K={k:5d} passes={cnt[k]:3d} us/pass={1e6 * agg[k] / cnt[k]:8.1f} total_ms={1e3 * agg[k]:7.2f}")
