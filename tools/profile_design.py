"""One full device-resident design (for ncu launch lists over a whole run)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_4711_b200 as vq
from paper_0910_4711_b200 import synthetic
from paper_0910_4711_b200.core import _Session
which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
spec = synthetic.WORKLOADS[which]
x = synthetic.make_training(which)
s = _Session(x, None)
conf = vq.LbgConfig(target_size=spec.target_size, epsilon=spec.epsilon, delta=spec.delta)
t0 = time.perf_counter(); cb, hist, warns, total, d, summ = s.train(conf); t1 = time.perf_counter()
print(which, "design", round(t1 - t0, 4), "s, passes", summ.passes)
