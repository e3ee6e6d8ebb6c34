"""Per-pass device time of the allocation pass (vqb_bench_assign: candidate
pass + re-rank + exact distances + distortion) at N=2^20, K=1024 for float32
rows vs float64 rows (not float32-exact) at L in {2, 5, 9, 16, 36}: the
float64 rows take the FP32 / tensor-core candidate pass on their rounded,
zero-padded copy with the rounding in the certified band."""
import ctypes, json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_0910_4711_b200 import _lib
from paper_0910_4711_b200.core import _Session

L = _lib.lib()
out = []
for dim in (2, 5, 9, 16, 36):
    rng = np.random.default_rng(100 + dim)
    x = rng.normal(0, 1, (1 << 20, dim)) * rng.uniform(0.5, 3.0, dim) + rng.uniform(-2, 2, dim)
    cb = np.ascontiguousarray(x[rng.choice(x.shape[0], 1024, replace=False)] + rng.normal(0, 0.05, (1024, dim)))
    row = {"dim": dim}
    for kind, s in (("f32", _Session(x.astype(np.float32), None)), ("f64", _Session(None, x))):
        ms, tot, fl = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        _lib.check(L.vqb_bench_assign(s.handle, _lib.ptr(cb), 1024, 3, ctypes.byref(ms), ctypes.byref(tot), ctypes.byref(fl)))
        _lib.check(L.vqb_bench_assign(s.handle, _lib.ptr(cb), 1024, 10, ctypes.byref(ms), ctypes.byref(tot), ctypes.byref(fl)))
        row[kind + "_ms"] = ms.value
        row[kind + "_flagged"] = fl.value
        row[kind + "_info"] = s.info()
        del s
    row["ratio_f64_over_f32"] = row["f64_ms"] / row["f32_ms"]
    out.append(row)
    print(json.dumps(row), flush=True)
