"""lbg_train from a float64 numpy matrix (what a reference user passes): cfg2."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_4711_b200 as vq
from paper_0910_4711_b200 import synthetic
x = synthetic.make_training("cfg2").astype(np.float64)
conf = vq.LbgConfig(target_size=1024, epsilon=1e-4, delta=0.01)
for rep in range(3):
    t0 = time.perf_counter(); ts = vq.TrainingSet(x); t1 = time.perf_counter()
    cb, st = vq.lbg_train(ts, conf); t2 = time.perf_counter()
    print(f"f64 rep{rep}: TrainingSet {t1 - t0:.4f}s lbg_train {t2 - t1:.4f}s total {t2 - t0:.4f}s", flush=True)
