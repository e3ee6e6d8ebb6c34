"""One cfg2 Lloyd iteration at K=1024 (the bench step; argv[2]: another K) for ncu captures:
session open, 2 warm-up passes + 1 profiled pass via vqb_bench_iteration."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_0910_4711_b200 import _lib, synthetic
from paper_0910_4711_b200.core import _Session

which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
g = np.load(os.path.join(ROOT, "tests", "golden", f"{which}_design.npz"))
cb = np.ascontiguousarray(g["cb"])
if len(sys.argv) > 2:  # a smaller codebook: the first K codevectors
    cb = np.ascontiguousarray(cb[: int(sys.argv[2])])
x = synthetic.make_training(which)
s = _Session(x, None)
segs = (ctypes.c_double * 5)()
fl = ctypes.c_int64()
for _ in range(3):
    _lib.check(_lib.lib().vqb_bench_iteration(s.handle, _lib.ptr(cb), cb.shape[0], 1, segs, ctypes.byref(fl)))
print(which, "segments ms", [round(v, 4) for v in segs], "flagged", fl.value)
