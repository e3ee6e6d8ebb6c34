import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import paper_0910_4711_b200 as vq
rng = np.random.default_rng(0)
cb = vq.Codebook(rng.uniform(0, 255, (1024, 16)))
for n in (1 << 12, 1 << 16, 1 << 20, 1 << 24):
    x = rng.uniform(0, 255, (n, 16)).astype(np.float32)
    vq.encode(x, cb)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); s = vq.encode(x, cb); ts.append(time.perf_counter() - t0)
    print(n, "encode from numpy: min %.3f ms, median %.3f ms" % (min(ts) * 1e3, sorted(ts)[2] * 1e3))
