"""Host-side profile of lbg_train from a numpy float32 matrix (cProfile, top entries)."""
import cProfile, os, pstats, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_4711_b200 as vq
from paper_0910_4711_b200 import synthetic

which = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
spec = synthetic.WORKLOADS[which]
x = synthetic.make_training(which)
conf = vq.LbgConfig(target_size=spec.target_size, epsilon=spec.epsilon, delta=spec.delta)
vq.lbg_train(vq.TrainingSet(x[: 1 << 14]), vq.LbgConfig(target_size=4))  # warm the library
for _ in range(2):
    t0 = time.perf_counter(); cb, st = vq.lbg_train(vq.TrainingSet(x), conf); t1 = time.perf_counter()
    print(which, "lbg_train from numpy:", round(t1 - t0, 4), "s")
pr = cProfile.Profile(); pr.enable()
cb, st = vq.lbg_train(vq.TrainingSet(x), conf)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
