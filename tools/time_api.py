"""Break down the host-API wall time of lbg_train / encode on the GPU box."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_4711_b200 as vq
from paper_0910_4711_b200 import synthetic
from paper_0910_4711_b200.core import _session_of
x = synthetic.make_training("cfg2")
spec = synthetic.WORKLOADS["cfg2"]
conf = vq.LbgConfig(target_size=spec.target_size, epsilon=spec.epsilon, delta=spec.delta)
for rep in range(3):
    t0 = time.perf_counter(); ts = vq.TrainingSet(x); t1 = time.perf_counter()
    s = _session_of(ts); t2 = time.perf_counter()
    cb, stats = vq.lbg_train(ts, conf); t3 = time.perf_counter()
    print(f"rep{rep}: TrainingSet {t1-t0:.4f}s  open+upload {t2-t1:.4f}s  train {t3-t2:.4f}s  total {t3-t0:.4f}s", flush=True)
cb5, q = synthetic.make_encode_case(n=1 << 24)
for rep in range(3):
    t0 = time.perf_counter(); st = vq.encode(q, vq.Codebook(cb5.astype(np.float64))); t1 = time.perf_counter()
    print(f"encode 2^24 rep{rep}: {t1-t0:.4f}s", flush=True)
