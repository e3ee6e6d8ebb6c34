"""Wall time of the public lbg_train on the cfg2 workload (host float32 in,
codebook out), several runs: the design's end-to-end cost incl. session
open / upload / row image / close."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_4711_b200 as vq
from paper_0910_4711_b200 import synthetic
which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
spec = synthetic.WORKLOADS[which]
x = synthetic.make_training(which)
conf = vq.LbgConfig(target_size=spec.target_size, epsilon=spec.epsilon, delta=spec.delta)
ts = []
for _ in range(4):
    t0 = time.perf_counter()
    ts_ = vq.TrainingSet(x)
    t1 = time.perf_counter()
    cb, st = vq.lbg_train(ts_, conf)
    ts.append((round(t1 - t0, 4), round(time.perf_counter() - t1, 4)))
print(which, "trainingset_s, lbg_train_s:", ts)
