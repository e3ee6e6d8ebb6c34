"""Pin the CPU oracle (oracle/) before trusting it: the reference's own
known-answer tests, and golden vectors produced by running the reference
(tests/golden/make_golden.py).  CPU only."""

import math
import os

import numpy as np
import pytest

import cases
import oracle
from conftest import GOLDEN


# ---------------------------------------------------------------------------
# reference KATs (pkg/tests/conftest.py, test_core.py, test_parallel.py)
# ---------------------------------------------------------------------------

TRACE = np.array([[0.0, 0.0], [0.0, 1.0], [4.0, 0.0], [4.0, 1.0]])
TRACE_SPLIT = np.array([[2.5, 1.0], [1.5, 0.0]])


def test_kat_trace_design():
    # test_core.py:340-347
    r = oracle.lbg_train(TRACE, 2, epsilon=1e-3, delta=0.5)
    assert r.codebook.tolist() == [[4.0, 0.5], [0.0, 0.5]]
    assert r.total == 1.0
    assert [(s, i, td) for s, i, td, _ in r.history] == [(2, 1, 11.0), (2, 2, 1.0), (2, 3, 1.0)]
    assert r.total / 4 == 0.25


def test_kat_trace_euclidean():
    # test_core.py:431-437
    r = oracle.lbg_train(TRACE, 2, delta=0.5, metric="euclidean")
    assert sorted(r.codebook.tolist()) == [[0.0, 0.5], [4.0, 0.5]]
    assert r.total == 2.0


def test_kat_split_and_assign():
    # test_core.py:192-201, 219-222
    assert oracle.split_rows(np.array([[2.0, 0.5]]), 0.5).tolist() == TRACE_SPLIT.tolist()
    assert oracle.split_rows(np.array([[0.0, 0.0], [4.0, 4.0]]), 0.01).tolist() == [
        [0.01, 0.01], [-0.01, -0.01], [4.01, 4.01], [3.99, 3.99]]
    cells, d = oracle.assign_cells(TRACE, TRACE_SPLIT)
    assert cells.tolist() == [1, 1, 0, 0] and d == 11.0


def test_kat_tie_rule_and_nearest():
    # test_core.py:157-165
    cells, dists = oracle.assign_all(np.array([[0.0, 0.0]]),
                                     np.array([[9.0, 9.0], [1.0, 0.0], [-1.0, 0.0]]))
    assert (cells[0], dists[0]) == (1, 1.0)
    cells, dists = oracle.assign_all(np.array([[1.0, 1.0]]), np.array([[0.0, 0.0], [5.0, 5.0]]))
    assert (cells[0], dists[0]) == (0, 2.0)


def test_kat_parallel_partials():
    # test_parallel.py:100-105: per-worker distortions [5.5, 5.5]
    cells, dists = oracle.assign_all(TRACE, TRACE_SPLIT, workers=2)
    parts = [oracle.sum_inorder(dists[lo:hi]) for lo, hi in oracle.partition_training(4, 2)]
    assert cells.tolist() == [1, 1, 0, 0] and parts == [5.5, 5.5]


def test_kat_update_and_empty():
    # test_core.py:265-285
    cb, empty = oracle.update_codebook(TRACE, np.array([1, 1, 0, 0]), TRACE_SPLIT)
    assert cb.tolist() == [[4.0, 0.5], [0.0, 0.5]] and empty == 0
    cb, empty = oracle.update_codebook(TRACE, np.array([0, 0, 0, 0]), TRACE_SPLIT)
    assert cb[0].tolist() == [2.0, 0.5] and cb[1].tolist() == [1.5, 0.0] and empty == 1


def test_kat_degenerate_and_target_one_and_guard():
    v = np.array([2.5, -1.5])
    r = oracle.lbg_train(np.tile(v, (5, 1)), 2, delta=0.5)
    assert r.codebook[0].tolist() == v.tolist() and r.codebook[1].tolist() == (v - 0.5).tolist()
    assert r.total == 0.0 and [h[3] for h in r.history] == [1, 1, 0]
    r = oracle.lbg_train(TRACE, 1)
    assert r.codebook.tolist() == [[2.0, 0.5]] and r.history == [] and r.total > 0
    rng = np.random.default_rng(29)
    r = oracle.lbg_train(rng.random((64, 3)), 8, epsilon=0.0, max_iterations_per_level=1)
    assert r.codebook.shape[0] == 8 and len(r.warnings) == 3
    assert all("1 iterations" in w for w in r.warnings)


def test_kat_convergence():
    # test_core.py:303-318
    assert oracle.convergence_check(100.0, 99.99, 1e-3) is True
    assert oracle.convergence_check(math.inf, 123.0, 1e-3) is False
    assert oracle.convergence_check(11.0, 1.0, 1e-3) is False
    assert oracle.convergence_check(0.0, 0.0, 0.0) is True
    assert oracle.convergence_check(10.0, 11.0, 0.0) is True


def test_partition_kats():
    # test_parallel.py:35-56
    sizes = lambda m, p: [hi - lo for lo, hi in oracle.partition_training(m, p)]
    assert sizes(2000, 4) == [500] * 4
    assert sizes(10, 4) == [3, 3, 2, 2]
    assert sizes(3, 5) == [1, 1, 1, 0, 0]


def test_pair_distance_and_centroid():
    assert oracle.pair_distance([0, 0], [3, 4], "euclidean") == 5.0
    assert oracle.pair_distance([0, 0], [3, 4], 0) == 25.0
    assert (oracle.column_sums(TRACE) / 4).tolist() == [2.0, 0.5]


# ---------------------------------------------------------------------------
# golden vectors produced by the reference itself
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("i", range(len(cases.assign_cases())))
def test_golden_assign(golden_small, i):
    case = cases.assign_cases()[i]
    cells, dists = oracle.assign_all(case["x"], case["cb"], case["metric"], workers=3)
    assert np.array_equal(cells, golden_small[f"assign{i}_cells"])
    assert dists.tobytes() == golden_small[f"assign{i}_dists"].tobytes()
    assert oracle.sum_inorder(dists) == float(golden_small[f"assign{i}_total"])


@pytest.mark.parametrize("i", range(len(cases.update_cases())))
@pytest.mark.parametrize("workers", [1, 3])
def test_golden_update(golden_small, i, workers):
    case = cases.update_cases()[i]
    new, counts = oracle.update_all(case["x"], case["cells"], case["cb"], workers)
    assert new.tobytes() == golden_small[f"update{i}_cb"].tobytes()
    assert np.array_equal(counts, golden_small[f"update{i}_counts"])


@pytest.mark.parametrize("i", range(len(cases.design_cases())))
def test_golden_design(golden_small, i):
    case = cases.design_cases()[i]
    cfg = dict(case["config"])
    metric = cfg.pop("distortion_metric", "squared_euclidean")
    target = cfg.pop("target_size")
    r = oracle.lbg_train(case["x"], target, metric=metric, **cfg)
    assert r.codebook.tobytes() == golden_small[f"design{i}_cb"].tobytes()
    hist = np.array(r.history, dtype=np.float64).reshape(-1, 4)
    assert hist.tobytes() == golden_small[f"design{i}_hist"].tobytes()
    assert r.total == float(golden_small[f"design{i}_total"])
    assert r.per_worker == golden_small[f"design{i}_per_worker"].tolist()
    assert len(r.warnings) == int(golden_small[f"design{i}_nwarn"])


@pytest.mark.parametrize("i", range(len(cases.encode_cases())))
def test_golden_encode(golden_small, i):
    case = cases.encode_cases()[i]
    idx = oracle.encode(case["x"], case["cb"], workers=case["workers"])
    assert idx.dtype == np.uint32
    assert np.array_equal(idx, golden_small[f"encode{i}_idx"])


def _design_golden(cfg):
    path = os.path.join(GOLDEN, f"{cfg}_design.npz")
    if not os.path.exists(path):
        pytest.skip(f"{cfg} golden not generated")
    return np.load(path)


def test_golden_cfg1_full_design():
    """cfg1 (BASELINE configs[0], the reference's CPU-runnable case): the whole
    design, bit for bit, including every pass's cell counts."""
    from paper_0910_4711_b200 import synthetic
    g = _design_golden("cfg1")
    spec = synthetic.WORKLOADS["cfg1"]
    x = synthetic.make_training("cfg1")
    import hashlib
    assert hashlib.sha256(x.tobytes()).hexdigest() == g["x_sha256"].item().decode()
    r = oracle.lbg_train(x.astype(np.float64), spec.target_size, epsilon=spec.epsilon,
                         delta=spec.delta, workers=4, record=True)
    assert r.codebook.tobytes() == g["cb"].tobytes()
    assert np.array(r.history, dtype=np.float64).tobytes() == g["hist"].tobytes()
    counts = np.concatenate([p.counts for p in r.passes]).astype(np.int32)
    assert np.array_equal(counts, g["pass_counts"])
