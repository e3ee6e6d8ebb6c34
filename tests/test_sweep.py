"""GPU sweep harness (paper_0910_4711_b200/sweep.py) on CPU: the Amdahl model,
the CSV and report formats of the reference's bench.py (pkg/tests/test_bench.py
is the model), and the P > 1 sweep protocol with gloo world 2 over the
EmulatedShard stand-in of tests/test_distributed.py."""

import numpy as np
import pytest

from paper_0910_4711_b200 import UsageError
from paper_0910_4711_b200 import sweep


def test_amdahl():
    assert sweep.amdahl_speedup(sweep.AmdahlParams(0.0, 8)) == 8.0
    assert sweep.amdahl_speedup(sweep.AmdahlParams(1.0, 8)) == 1.0
    assert sweep.amdahl_speedup(sweep.AmdahlParams(0.15, 4)) == pytest.approx(1 / (0.15 + 0.85 / 4))
    with pytest.raises(UsageError):
        sweep.AmdahlParams(1.5, 2)
    with pytest.raises(UsageError):
        sweep.AmdahlParams(0.1, 0)


def test_synthetic_set_is_the_reference_generator():
    ts = sweep.synthetic_training_set(100, 10, 42)
    assert ts.vectors.tobytes() == np.random.default_rng(42).random((100, 10)).tobytes()


def test_csv_and_report(tmp_path):
    recs = [sweep.BenchRecord(8, 1, 2000, 10, 0.5, 12.25, 7),
            sweep.BenchRecord(8, 2, 2000, 10, 0.25, 12.25, 7)]
    path = tmp_path / "b.csv"
    sweep.write_bench_csv(recs, path, comment="gpu sweep")
    assert path.read_text() == ("# gpu sweep\nn,p,m,k,seconds,td,iterations\n"
                                "8,1,2000,10,0.5,12.25,7\n8,2,2000,10,0.25,12.25,7\n")
    lines = sweep.speedup_report(recs)
    assert lines[1] == ("N=8 P=2: measured speedup 2.00x, Amdahl prediction 1.74x "
                        "(serial fraction 0.15)")


def test_sweep_validates():
    ts = sweep.synthetic_training_set(10, 2, 1)
    with pytest.raises(UsageError):
        sweep.run_sweep(ts, repeats=0)
    with pytest.raises(UsageError):
        sweep.run_sweep(ts, gpu_counts=(0,))


@pytest.mark.timeout(600)
def test_world2_sweep_over_gloo_matches_world1():
    """P = 1 and P = 2 columns of the sweep through the spawned-rank protocol
    (gloo, EmulatedShard): same designs bit for bit, reference cell order."""
    x = np.random.default_rng(7).integers(0, 256, (4096 + 512, 4)).astype(np.float32)
    ts = sweep.TrainingSet(x)
    recs = sweep.run_sweep(ts, sizes=(4, 8), gpu_counts=(1, 2), repeats=1, backend="gloo",
                           backend_factory="test_distributed:EmulatedShard")
    assert [(r.codebook_size, r.workers) for r in recs] == [(4, 1), (4, 2), (8, 1), (8, 2)]
    for a, b in zip(recs[0::2], recs[1::2]):
        assert (a.td, a.iterations) == (b.td, b.iterations)
        assert a.vector_count == 4608 and a.dimension == 4 and a.seconds > 0
    assert len(sweep.speedup_report(recs)) == 4
