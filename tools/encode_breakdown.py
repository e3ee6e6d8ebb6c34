"""Where the time of a cfg5-sized encode() from pageable numpy goes: the same
vqb_encode_f32 call with a fresh (never touched) and a pre-touched output
array, and with a pinned input."""
import ctypes, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0910_4711_b200 import _lib
import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
rng = np.random.default_rng(0)
cb = np.ascontiguousarray(rng.uniform(0, 255, (1024, 16)))
x = (rng.random((n, 16), dtype=np.float32) * np.float32(255.0))
L = _lib.lib()

def call(xa, out):
    t0 = time.perf_counter()
    _lib.check(L.vqb_encode_f32(_lib.ptr(xa), n, 16, _lib.ptr(cb), 1024, 0, _lib.ptr(out), None))
    return time.perf_counter() - t0

out = np.empty(n, dtype=np.uint32); call(x, out)
for label, fresh in (("fresh output", True), ("touched output", False), ("fresh output", True), ("touched output", False)):
    o = np.empty(n, dtype=np.uint32) if fresh else out
    print(f"pageable input, {label}: {call(x, o) * 1e3:.1f} ms")
xp = torch.from_numpy(x).pin_memory().numpy()
for label, fresh in (("fresh output", True), ("touched output", False)):
    o = np.empty(n, dtype=np.uint32) if fresh else out
    print(f"pinned input, {label}: {call(xp, o) * 1e3:.1f} ms")
op = torch.empty(n, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
print(f"pinned input, pinned output: {call(xp, op) * 1e3:.1f} ms")
