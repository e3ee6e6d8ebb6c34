"""Time the device mixture generator at cfg4 / cfg5 sizes (vqb_open_gmm:
generation + column statistics + session setup) against the host numpy
generator + upload it replaces.  Prints one JSON line per case."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_0910_4711_b200 import synthetic  # noqa: E402

for cfg in sys.argv[1:] or ["cfg4", "cfg5"]:
    spec = synthetic.WORKLOADS[cfg]
    synthetic.make_training_device(cfg, 1 << 16)  # warm
    t = []
    for _ in range(3):
        t0 = time.perf_counter()
        ts, _ = synthetic.make_training_device(cfg)
        t.append(time.perf_counter() - t0)
        del ts
    t0 = time.perf_counter()
    x = synthetic.make_training(cfg) if cfg != "cfg5" else synthetic.make_encode_case()[1]
    host = time.perf_counter() - t0
    print(json.dumps({"cfg": cfg, "rows": spec.n, "device_open_s": min(t), "host_numpy_s": host,
                      "bytes": int(x.nbytes)}), flush=True)
