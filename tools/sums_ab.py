"""A/B of the cell-sum kernels: per-kernel segments of one Lloyd iteration
(vqb_bench_iteration) for cfg2 / cfg3 / cfg4 at their converged codebooks.
Usage: VQB_SUMS_RED=0|1 python tools/sums_ab.py cfg2 cfg4 ..."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_0910_4711_b200 import _lib, synthetic
from paper_0910_4711_b200.core import _Session

for which in sys.argv[1:]:
    g = np.load(os.path.join(ROOT, "tests", "golden", f"{which}_design.npz"))
    x = synthetic.make_training(which)
    s = _Session(x, None)
    segs = (ctypes.c_double * 5)()
    fl = ctypes.c_int64()
    for k in [int(v) for v in os.environ.get("KS", "0,256,64").split(",")]:
        k = k or g["cb"].shape[0]
        cb = np.ascontiguousarray(g["cb"][:k])
        acc = np.zeros(5)
        for r in range(8):
            _lib.check(_lib.lib().vqb_bench_iteration(s.handle, _lib.ptr(cb), k, 1, segs, ctypes.byref(fl)))
            if r >= 3:
                acc += np.array(list(segs))
        print(which, "K", k, "segments ms [stage, assign, rerank, epilogue, finalize]",
              [round(v, 4) for v in acc / 5], "flagged", fl.value, flush=True)
    del s
