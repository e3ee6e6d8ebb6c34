"""Validate the tcgen05 candidate pass on the GPU: raw TMEM accumulators of
one 128-row tile vs the float64 emulation of the same fp16 operands."""
import ctypes, json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_0910_4711_b200 import _lib, synthetic
from paper_0910_4711_b200.core import _Session
import tc_emulation as te

out = {}
for name, (x, cb) in {
    "cfg2_L16_K1024": (synthetic.make_training("cfg2", n=4096), np.load(os.path.join(ROOT, "tests/golden/cfg2_design.npz"))["cb"]),
    "cfg3_L64_K512": (synthetic.make_training("cfg3", n=65536)[:4096], np.load(os.path.join(ROOT, "tests/golden/cfg3_design.npz"))["cb"]),
    "rand_L32_K256": (np.random.default_rng(1).normal(50, 30, (4096, 32)).astype(np.float32),
                      np.random.default_rng(2).normal(50, 30, (256, 32))),
}.items():
    s = _Session(np.ascontiguousarray(x), None)
    K = cb.shape[0]
    dump = np.empty((128, K), dtype=np.float32)
    sc = np.zeros(5, dtype=np.int32)
    _lib.check(_lib.lib().vqb_debug_tc_tile(s.handle, _lib.ptr(np.ascontiguousarray(cb)), K, _lib.ptr(dump), _lib.ptr(sc)))
    ey, ew, kn = int(sc[0]), int(sc[1]), int(sc[2])
    mu = te.session_mu(x)
    d, mag, v = te.expected_accumulators(x[:128], mu, cb, ey, ew, kn)
    err = np.abs(dump.astype(np.float64) - d)
    rel = err / mag
    L = x.shape[1]
    out[name] = {"scales": sc.tolist(), "max_err_over_mag": float(rel.max()), "p99": float(np.quantile(rel, 0.99)),
                 "bound": (3 * L + 2) * 2.0 ** -22, "max_abs_err": float(err.max()),
                 "split_err_vs_exact_over_mag": float((np.abs(d - v) / mag).max()),
                 "argmin_agree_frac": float(np.mean(np.argmin(dump, 1) == np.argmin(v, 1)))}
print(json.dumps(out, indent=1))
