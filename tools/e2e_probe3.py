import ctypes, os, sys, time, statistics
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0910_4711_b200 import _lib, synthetic
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
    return [round(t * 1e3, 2) for t in ts]
d = torch.empty(n * 16, dtype=torch.float32, device="cuda")
def h2d(t, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(t.view(-1), non_blocking=True); torch.cuda.synchronize(); ts.append(round((time.perf_counter() - t0) * 1e3, 3))
    return ts
print("warm lib", e2e(torch.from_numpy(x).pin_memory().numpy(), 3))
for k in range(4):
    t = torch.from_numpy(x).pin_memory()
    print(f"buf{k} h2d", h2d(t), "e2e", e2e(t.numpy()), flush=True)
    time.sleep(1.0)
    print(f"buf{k} after 1s h2d", h2d(t), "e2e", e2e(t.numpy()), flush=True)
