"""Host->device bandwidth of the copy engine (pageable staged, pinned, plain
cudaMemcpy, cudaHostRegister) for a 1 GiB buffer; one JSON line."""
import ctypes, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0910_4711_b200 import _lib
L = _lib.lib()
n = 1 << 30
a = np.random.default_rng(0).integers(0, 255, n, dtype=np.uint8)
pinned = torch.from_numpy(a.copy()).pin_memory().numpy()
out = {"cpus": os.cpu_count()}
for name, buf, mode in [("pageable_staged", a, 0), ("pageable_plain_memcpy", a, 1), ("pinned", pinned, 0),
                        ("host_register_then_upload", a, 2)]:
    best = 1e9
    for _ in range(3):
        sec = ctypes.c_double()
        _lib.check(L.vqb_bench_upload(buf.ctypes.data, n, mode, ctypes.byref(sec)))
        best = min(best, sec.value)
    out[name + "_GBps"] = round(n / best / 1e9, 2)
print(json.dumps(out))
