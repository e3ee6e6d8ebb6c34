"""Device-timestamp trace (VQB_TRACE=1) of the host-buffer Lloyd step at cfg4 from pinned memory."""
import ctypes, os, sys
os.environ["VQB_TRACE"] = "1"
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0910_4711_b200 import _lib, synthetic
which = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", f"{which}_design.npz"))
cb = np.ascontiguousarray(g["cb"]); K = cb.shape[0]
x = synthetic.make_training(which)
xp = torch.from_numpy(x).pin_memory().numpy()
new = np.empty_like(cb); td = ctypes.c_double(); ne = ctypes.c_int64()
L = _lib.lib()
for i in range(3):
    print(f"--- call {i}", file=sys.stderr)
    _lib.check(L.vqb_lloyd_step_f32(_lib.ptr(xp), x.shape[0], 16, _lib.ptr(cb), K, 0, _lib.ptr(new), None,
                                    ctypes.byref(td), ctypes.byref(ne)))
