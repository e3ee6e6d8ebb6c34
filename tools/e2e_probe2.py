"""e2e Lloyd step timing under the same process history as bench.py."""
import ctypes, os, sys, time, statistics
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0910_4711_b200 import _lib, synthetic
from paper_0910_4711_b200.core import _Session
L = _lib.lib()
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/cfg2_design.npz"))
cb = np.ascontiguousarray(g["cb"]); K = cb.shape[0]
x = synthetic.make_training("cfg2"); n = x.shape[0]
new = np.empty_like(cb); td = ctypes.c_double(); em = ctypes.c_int64()
def e2e(buf, reps=8):
    ts = []
    for i in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        _lib.check(L.vqb_lloyd_step_f32(_lib.ptr(buf), n, 16, _lib.ptr(cb), K, 0, _lib.ptr(new), None, ctypes.byref(td), ctypes.byref(em)))
        ts.append(time.perf_counter() - t0)
    return round(min(ts[2:]) * 1e3, 3), round(statistics.median(ts[2:]) * 1e3, 3)
xp = torch.from_numpy(x).pin_memory().numpy()
print("fresh", e2e(xp))
sess = _Session(x, None)
print("after session open", e2e(xp))
ops, sec = ctypes.c_double(), ctypes.c_double()
_lib.check(L.vqb_pipe_microbench(0, 4, 4000, ctypes.byref(ops), ctypes.byref(sec)))
print("after ffma microbench", e2e(xp))
segs = (ctypes.c_double * 5)(); fl = ctypes.c_int64()
for _ in range(13):
    _lib.check(L.vqb_bench_iteration(sess.handle, _lib.ptr(cb), K, 1, segs, ctypes.byref(fl)))
print("after bench iterations", e2e(xp))
xp2 = torch.from_numpy(x).pin_memory().numpy()
print("fresh pinned copy", e2e(xp2))
