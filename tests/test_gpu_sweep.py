"""GPU sweep harness on one B200: the P = 1 column of run_sweep designs the
reference's benchmark data (bench.py:59-62, 2000 x 10 uniform, seed 42) and
matches the oracle's design cell for cell.  GPU only."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

from paper_0910_4711_b200 import _lib, sweep  # noqa: E402


def test_single_gpu_sweep_matches_oracle(tmp_path):
    if _lib.device_count() < 1:
        pytest.fail("GPU tests need a CUDA device")
    ts = sweep.synthetic_training_set(2000, 10, 42)
    recs = sweep.run_sweep(ts, sizes=(8, 16, 32), gpu_counts=(1,), repeats=2)
    for r in recs:
        ref = oracle.lbg_train(ts.vectors, r.codebook_size, epsilon=1e-3, delta=0.01)
        assert r.iterations == len(ref.history)
        assert r.td == pytest.approx(ref.total, rel=1e-12)
        assert r.seconds > 0 and r.workers == 1
    sweep.write_bench_csv(recs, tmp_path / "sweep.csv")
    assert (tmp_path / "sweep.csv").read_text().startswith("n,p,m,k,seconds,td,iterations\n8,1,2000,10,")
    assert len(sweep.speedup_report(recs)) == 3
