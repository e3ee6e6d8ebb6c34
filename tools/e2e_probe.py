"""Time the host-buffer Lloyd step (vqb_lloyd_step_f32) and its pieces."""
import ctypes, os, sys, time, statistics
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0910_4711_b200 import _lib, synthetic
L = _lib.lib()
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/cfg2_design.npz"))
cb = np.ascontiguousarray(g["cb"]); K = cb.shape[0]
x = synthetic.make_training("cfg2"); n = x.shape[0]
xp_t = torch.from_numpy(x).pin_memory(); xp = xp_t.numpy()
new = np.empty_like(cb); td = ctypes.c_double(); em = ctypes.c_int64()
def step(buf):
    _lib.check(L.vqb_lloyd_step_f32(_lib.ptr(buf), n, 16, _lib.ptr(cb), K, 0, _lib.ptr(new), None, ctypes.byref(td), ctypes.byref(em)))
for name, buf in [("pinned", xp), ("pageable", x)]:
    ts = []
    for i in range(12):
        torch.cuda.synchronize(); t0 = time.perf_counter(); step(buf); ts.append(time.perf_counter() - t0)
    print(name, "ms: min %.3f med %.3f" % (min(ts[2:]) * 1e3, statistics.median(ts[2:]) * 1e3), [round(t * 1e3, 2) for t in ts])
d = torch.empty(n * 16, dtype=torch.float32, device="cuda")
ts = []
for i in range(10):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(xp_t.view(-1), non_blocking=True); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print("torch pinned H2D 64MB ms: min %.3f" % (min(ts) * 1e3))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
big = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for mode in ("zero", "zero+read"):
    ts = []
    for i in range(10):
        flush.zero_()
        if mode == "zero+read":
            big.sum()  # evicts the dirty lines (their write-back happens here)
        torch.cuda.synchronize(); t0 = time.perf_counter(); step(xp); ts.append(time.perf_counter() - t0)
    print("pinned after", mode, "ms: min %.3f med %.3f" % (min(ts[2:]) * 1e3, statistics.median(ts[2:]) * 1e3))
import subprocess
p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                      "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.DEVNULL)
time.sleep(0.5)
ts = []
for i in range(10):
    torch.cuda.synchronize(); t0 = time.perf_counter(); step(xp); ts.append(time.perf_counter() - t0)
p.terminate()
print("pinned with nvidia-smi -lms 20 running ms: min %.3f med %.3f" % (min(ts[2:]) * 1e3, statistics.median(ts[2:]) * 1e3), [round(t*1e3,2) for t in ts])
