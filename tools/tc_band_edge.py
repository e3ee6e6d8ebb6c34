"""Measured tcgen05 accumulation error against the certification band's budget
(2 x 2^-22 of the magnitude sum per MMA) on the band-edge operand sets of
tests/test_gpu_parity.py::test_tc_accumulators_band_edge_operands: one line
per case with max(err / budget)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests")); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import tc_emulation as te
from test_gpu_parity import _tc_edge_operands
from paper_0910_4711_b200 import _lib
from paper_0910_4711_b200.core import _Session

REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for kind in ("cancel", "signs", "ones", "range"):
    for dim, k in ((16, 4096), (16, 256), (32, 768), (64, 512), (64, 2048)):
        worst, samples = 0.0, 0
        for rep in range(REPS):  # the probe dumps the first 128-row tile: fresh draws per repetition
            rng = np.random.default_rng(sum(map(ord, kind)) * 1000003 + dim * 8191 + k + 7919 * rep)
            x, cb = _tc_edge_operands(kind, dim, k, rng)
            s = _Session(x, None)
            dump = np.empty((128, k), dtype=np.float32); sc = np.zeros(5, dtype=np.int32)
            _lib.check(_lib.lib().vqb_debug_tc_tile(s.handle, _lib.ptr(cb), k, _lib.ptr(dump), _lib.ptr(sc)))
            d, mag, v = te.expected_accumulators(x[:128], te.session_mu(x), cb, int(sc[0]), int(sc[1]), int(sc[2]))
            n_mma = 3 * dim // 16 + 1
            ratio = np.abs(dump.astype(np.float64) - d) / (2 * n_mma * 2.0 ** -22 * mag)
            worst = max(worst, float(ratio.max())); samples += ratio.size
        print(f"{kind:7s} L={dim:2d} K={k:4d} tc_on={sc[3]} bad={sc[4]} accumulators={samples} max err/budget = {worst:.4f}")
