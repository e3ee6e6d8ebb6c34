"""Parity depth, round 2 (GPU only): the two-word fixed-point cell sums and
their exactness detector, the reference-order fallback, every public entry
point, teacher forcing on cfg4 and per-pass centroids, non-finite query rows,
history beyond the device ring, and threads sharing a TrainingSet.

Reference citations: _kernels.py:18-98 (kernels), core.py:235-339 (entry
points), parallel.py:157-253 (parallel_assign / integrate / parallel_update),
codec.py:62-93 (encode)."""

import math
import os
import subprocess
import sys
import threading

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu

vq = pytest.importorskip("paper_0910_4711_b200")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    from paper_0910_4711_b200 import _lib
    if _lib.device_count() < 1:
        pytest.fail("GPU tests need a CUDA device")


def _golden(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{name} golden not generated")
    return np.load(path)


def _lowbit(v: float) -> int:
    if v == 0.0:
        return 2**31 - 1
    m, e = math.frexp(abs(v))
    q = int(m * 2**53)
    return e - 53 + ((q & -q).bit_length() - 1)


def _hetero(n, dim=16, seed=11):
    """float32 rows whose columns span 1e3 .. 1e-4 (and one 1e6 column)."""
    rng = np.random.default_rng(seed)
    scales = np.array([1e3, 1e-4, 1.0, 1e6, 3e-2, 250.0, 1e-3, 7.0] * (dim // 8 + 1))[:dim]
    x = rng.normal(0.0, 1.0, (n, dim)) * scales + rng.uniform(-2, 2, dim) * scales
    return x.astype(np.float32)


def _exact_where_different(got, want, x, cells, k, cap=300):
    """Where the reference's ascending-order FP64 cell sum rounded (long
    cells, tiny coordinates beside large ones) the device centroid is the
    EXACT cell sum rounded once, divided by the count: check every differing
    entry (up to `cap`) against math.fsum (the correctly rounded exact sum).
    Returns the number of differing entries."""
    diff = np.argwhere(got != want)
    x64 = np.asarray(x, dtype=np.float64)
    order = np.argsort(cells, kind="stable")
    bounds = np.searchsorted(cells[order], np.arange(k + 1))
    for c, l in diff[:cap]:
        members = x64[order[bounds[c]:bounds[c + 1]], l]
        assert got[c, l] == math.fsum(members.tolist()) / float(len(members)), (c, l)
    return len(diff)


def _rel(a, b):
    den = np.maximum(np.abs(b), 1e-300)
    return float(np.max(np.abs(a - b) / den))


# ---------------------------------------------------------------------------
# column stats and the fixed-point plan
# ---------------------------------------------------------------------------

def test_colstats_match_numpy():
    x = _hetero(5000, 16)
    x[:, 5] = 0.0
    from paper_0910_4711_b200.core import _Session
    s = _Session(x, None)
    cmax, clow = s.colstats()
    assert np.array_equal(cmax, np.max(np.abs(x.astype(np.float64)), axis=0))
    want = [min(_lowbit(float(v)) for v in col) for col in x.astype(np.float64).T]
    assert clow.tolist() == want


# ---------------------------------------------------------------------------
# heterogeneous column scales: the per-column two-word grid keeps every
# coordinate exact, so the centroids are the exact cell means rounded once
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("n", [1 << 20, 1 << 24])
def test_heterogeneous_columns_update_vs_oracle(n):
    dim = 16 if n <= (1 << 20) else 8
    x = _hetero(n, dim)
    rng = np.random.default_rng(n)
    k = 256
    cb = rng.normal(0, 1, (k, dim)) * np.max(np.abs(x), axis=0)
    cells = rng.integers(0, k - 3, n)  # the last 3 cells stay empty
    ts = vq.TrainingSet(x)
    new, empty = vq.update_codebook(ts, vq.CellTable(cells, k), vq.Codebook(cb))
    want, want_empty = oracle.update_codebook(x.astype(np.float64), cells, cb)
    assert empty == want_empty == 3
    rel = _rel(new.codevectors, want)
    assert rel <= 1e-12, rel  # north star: 1e-5
    ndiff = _exact_where_different(new.codevectors, want, x, cells, k)
    assert ndiff <= 0.5 * want.size, ndiff
    # the empty cells keep their rows bit for bit
    assert new.codevectors[k - 3:].tobytes() == cb[k - 3:].tobytes()


def test_heterogeneous_columns_design_vs_oracle():
    n = 1 << 20
    x = _hetero(n, 16)
    conf = vq.LbgConfig(target_size=16, epsilon=1e-4, delta=0.01)
    cb, stats = vq.lbg_train(vq.TrainingSet(x), conf)
    ref = oracle.lbg_train(x.astype(np.float64), 16, epsilon=1e-4, delta=0.01,
                           workers=oracle.max_threads())
    got = [(h.codebook_size, h.iteration, h.empty_cells) for h in stats.history]
    assert got == [(s, i, e) for s, i, _, e in ref.history]
    np.testing.assert_allclose([h.td for h in stats.history], [h[2] for h in ref.history],
                               rtol=1e-12)
    assert _rel(cb.codevectors, ref.codebook) <= 1e-12


def test_outlier_exact_fixed_point():
    """U(0, 1e-3) with one 1e6 outlier (the advisor's case): the two-word grid
    stays exact, so no centroid collapses and all agree with the oracle."""
    rng = np.random.default_rng(2)
    x = rng.uniform(0, 1e-3, (1 << 16, 4)).astype(np.float32)
    x[77, 2] = 1e6
    ts = vq.TrainingSet(x)
    from paper_0910_4711_b200.core import _session_of
    k = 64
    cb = rng.uniform(0, 1e-3, (k, 4))
    cells = rng.integers(0, k, x.shape[0])
    new, _ = vq.update_codebook(ts, vq.CellTable(cells, k), vq.Codebook(cb))
    want, _ = oracle.update_codebook(x.astype(np.float64), cells, cb)
    assert _rel(new.codevectors, want) <= 1e-12
    _exact_where_different(new.codevectors, want, x, cells, k)
    conf = vq.LbgConfig(target_size=8, epsilon=1e-3, delta=1e-5)
    out = _session_of(ts).train(conf)
    summ = out[5]
    assert summ.sums_exact == 1 and summ.ordered == 0
    ref = oracle.lbg_train(x.astype(np.float64), 8, epsilon=1e-3, delta=1e-5)
    assert [(h.codebook_size, h.iteration, h.empty_cells) for h in out[1]] == \
        [(s, i, e) for s, i, _, e in ref.history]
    assert _rel(out[0], ref.codebook) <= 1e-12


def test_outlier_beyond_grid_takes_reference_order():
    """A finite 1e30 outlier beside 1e-3 values: no two-word grid holds the
    column, the detector fires and the reference-order sums run -- results
    bit-identical to the reference's (previously every small centroid
    collapsed to 0)."""
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1e-3, (1 << 16, 4)).astype(np.float32)
    x[123, 1] = np.float32(1e30)
    ts = vq.TrainingSet(x)
    from paper_0910_4711_b200.core import _session_of
    k = 32
    cb = rng.uniform(0, 1e-3, (k, 4))
    cells = rng.integers(0, k, x.shape[0])
    new, _ = vq.update_codebook(ts, vq.CellTable(cells, k), vq.Codebook(cb))
    want, _ = oracle.update_codebook(x.astype(np.float64), cells, cb)
    assert new.codevectors.tobytes() == want.tobytes()
    conf = vq.LbgConfig(target_size=8, epsilon=1e-3, delta=1e-5)
    out = _session_of(ts).train(conf)
    assert out[5].sums_exact == 0 and out[5].ordered == 1
    ref = oracle.lbg_train(x.astype(np.float64), 8, epsilon=1e-3, delta=1e-5)
    assert [(h.codebook_size, h.iteration, h.td, h.empty_cells) for h in out[1]] == ref.history
    assert out[0].tobytes() == ref.codebook.tobytes()


def test_float64_rows_reference_order_bit_identical():
    """float64 rows float32 cannot hold: the reference-order path (stable
    counting sort + sequential FP64 chains) reproduces update_rows and the
    whole design bit for bit."""
    rng = np.random.default_rng(4)
    x = rng.normal(0, 1, (30000, 5)) * np.array([1.0, 10.0, 1e-2, 3.0, 100.0])
    k = 48
    cb = rng.normal(0, 1, (k, 5))
    cells = rng.integers(0, k, x.shape[0])
    ts = vq.TrainingSet(x)
    new, _ = vq.update_codebook(ts, vq.CellTable(cells, k), vq.Codebook(cb))
    want, _ = oracle.update_codebook(x, cells, cb)
    assert new.codevectors.tobytes() == want.tobytes()
    conf = vq.LbgConfig(target_size=16, epsilon=1e-3, delta=0.01)
    cbk, stats = vq.lbg_train(ts, conf)
    ref = oracle.lbg_train(x, 16, epsilon=1e-3, delta=0.01)
    assert stats.td_history() == [(s, i, td) for s, i, td, _ in ref.history]
    assert cbk.codevectors.tobytes() == ref.codebook.tobytes()


# ---------------------------------------------------------------------------
# every public entry point
# ---------------------------------------------------------------------------

def test_nearest_codevector_kats_and_oracle():
    cb = vq.Codebook(np.array([[9.0, 9.0], [1.0, 0.0], [-1.0, 0.0]]))
    assert vq.nearest_codevector([0.0, 0.0], cb) == (1, 1.0)  # tie -> lowest index
    assert vq.nearest_codevector([0.0, 0.0], cb, metric="euclidean") == (1, 1.0)
    dup = vq.Codebook(np.array([[1.0, 1.0], [1.0, 1.0], [0.0, 5.0]]))
    assert vq.nearest_codevector([1.0, 1.0], dup) == (0, 0.0)
    rng = np.random.default_rng(6)
    big = rng.normal(0, 1, (1000, 16))
    book = vq.Codebook(big)
    for q in rng.normal(0, 1, (50, 16)):
        cells, dists = oracle.assign_all(q.reshape(1, -1), big)
        assert vq.nearest_codevector(q, book) == (int(cells[0]), float(dists[0]))
    with pytest.raises(vq.UsageError):
        vq.nearest_codevector([0.0, 1.0, 2.0], cb)
    with pytest.raises(vq.UsageError):
        vq.nearest_codevector([0.0, float("nan")], cb)


def test_centroid_and_distance_vs_oracle():
    rng = np.random.default_rng(7)
    x = rng.normal(0, 1, (3001, 7))
    assert vq.centroid(x).tobytes() == (oracle.column_sums(x) / x.shape[0]).tobytes()
    assert vq.centroid(vq.TrainingSet(x)).tobytes() == (oracle.column_sums(x) / 3001).tobytes()
    x32 = rng.uniform(0, 255, (4096, 16)).astype(np.float32)
    want = oracle.column_sums(x32.astype(np.float64)) / 4096
    assert vq.centroid(vq.TrainingSet(x32)).tobytes() == want.tobytes()
    assert vq.centroid([[1.0, 2.0], [3.0, 5.0]]).tolist() == [2.0, 3.5]
    with pytest.raises(vq.DomainError):
        vq.centroid([])
    a, b = rng.normal(0, 1, 13), rng.normal(0, 1, 13)
    assert vq.distance(a, b) == oracle.pair_distance(a, b, 0)
    assert vq.distance(a, b, "euclidean") == oracle.pair_distance(a, b, 1)
    assert vq.distance([0, 0], [3, 4], "euclidean") == 5.0
    with pytest.raises(vq.UsageError):
        vq.distance([0, 0], [1, 2, 3])


def test_parallel_assign_integrate_update_vs_oracle():
    rng = np.random.default_rng(8)
    x = rng.normal(0, 1, (10007, 16)).astype(np.float32)
    cb = rng.normal(0, 1, (128, 16))
    ts, book = vq.TrainingSet(x), vq.Codebook(cb)
    cells, dists = oracle.assign_all(x.astype(np.float64), cb)
    for workers in (1, 3, 8):
        plan = vq.partition_training(ts.m, workers)
        partials, dist = vq.parallel_assign(ts, book, plan)
        assert [p.start for p in partials] == [lo for lo, _ in plan.ranges]
        for p, (lo, hi) in zip(partials, plan.ranges):
            assert np.array_equal(p.cells, cells[lo:hi])
        assert dist == [oracle.sum_inorder(dists[lo:hi]) for lo, hi in plan.ranges]
        table, total = vq.integrate(partials, dist)
        assert np.array_equal(table.cells, cells)
        want_total = 0.0
        for d in dist:
            want_total += d
        assert total == want_total
        new, empty = vq.parallel_update(ts, table, book, workers)
        want, want_empty = oracle.update_codebook(x.astype(np.float64), cells, cb)
        assert new.codevectors.tobytes() == want.tobytes() and empty == want_empty
    with pytest.raises(vq.InternalError):
        vq.integrate(partials[::-1], dist[::-1])
    with pytest.raises(vq.UsageError):
        vq.parallel_assign(ts, book, vq.partition_training(ts.m + 1, 2))


# ---------------------------------------------------------------------------
# teacher forcing: cfg4 counts, per-pass centroids on cfg1-4
# ---------------------------------------------------------------------------

def test_teacher_forced_counts_cfg4():
    from paper_0910_4711_b200 import synthetic
    g = _golden("cfg4_design")
    ts = vq.TrainingSet(synthetic.make_training("cfg4"))
    counts = g["pass_counts"]
    offs = np.cumsum([0] + [int(s) for s in g["hist"][:, 0]])
    checked = 0
    for p in range(len(offs) - 1):
        key = f"pass{p}_cb"
        if key not in g.files:
            continue
        table, _ = vq.assign_cells(ts, vq.Codebook(g[key]))
        got = np.bincount(table.cells, minlength=g[key].shape[0])
        assert np.array_equal(got, counts[offs[p]:offs[p + 1]]), p
        checked += 1
    assert checked >= 100


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_teacher_forced_centroids(cfg):
    """Pass p's recorded codebook -> our allocation + update == pass p+1's
    recorded codebook (same level; 1e-5 is the north star, the sums are
    exact), and a converged level's split is bit-exact."""
    from paper_0910_4711_b200 import synthetic
    g = _golden(f"{cfg}_design")
    ts = vq.TrainingSet(synthetic.make_training(cfg))
    hist = g["hist"]
    keys = sorted(int(k[4:-3]) for k in g.files if k.startswith("pass") and k.endswith("_cb"))
    pairs = same = split = 0
    worst = 0.0
    for p in keys:
        if p + 1 not in keys:
            continue
        cb0, cb1 = g[f"pass{p}_cb"], g[f"pass{p + 1}_cb"]
        if cb1.shape[0] == cb0.shape[0]:
            table, _ = vq.assign_cells(ts, vq.Codebook(cb0))
            new, _ = vq.update_codebook(ts, table, vq.Codebook(cb0))
            worst = max(worst, _rel(new.codevectors, cb1))
            same += int(new.codevectors.tobytes() == cb1.tobytes())
            pairs += 1
        elif int(hist[p, 1]) < 100:  # converged -> plain split of the same codebook
            assert vq.split_codebook(vq.Codebook(cb0), float(synthetic.WORKLOADS[cfg].delta)) \
                .codevectors.tobytes() == cb1.tobytes()
            split += 1
    assert pairs >= 5 and split >= 1
    assert worst <= 1e-5, worst
    if cfg in ("cfg1", "cfg3"):  # 8-bit pixels: the reference's sums are exact too
        assert same == pairs


# ---------------------------------------------------------------------------
# non-finite query rows (raw matrices skip TrainingSet's check)
# ---------------------------------------------------------------------------

def test_nonfinite_rows_encode_and_assign_cells():
    rng = np.random.default_rng(9)
    x = rng.normal(0, 1, (5000, 16))
    bad = [3, 1000, 4999]
    x[3, 5] = np.nan
    x[1000, 0] = np.inf
    x[4999, 15] = -np.inf
    cb = rng.normal(0, 1, (256, 16))
    cells, dists = oracle.assign_all(x, cb)
    assert cells[bad].tolist() == [0, 0, 0] and np.all(np.isinf(dists[bad]))
    stream = vq.encode(x, vq.Codebook(cb))
    assert np.array_equal(stream.indices, cells.astype(np.uint32))
    stream32 = vq.encode(x.astype(np.float32), vq.Codebook(cb))
    cells32, _ = oracle.assign_all(x.astype(np.float32).astype(np.float64), cb)
    assert np.array_equal(stream32.indices, cells32.astype(np.uint32))
    table, total = vq.assign_cells(x, vq.Codebook(cb))
    assert np.array_equal(table.cells, cells) and total == math.inf
    with pytest.raises(vq.UsageError):
        vq.TrainingSet(x)


# ---------------------------------------------------------------------------
# history: any number of records (the device ring is drained per batch)
# ---------------------------------------------------------------------------

def test_history_longer_than_the_device_ring():
    code = (
        "import sys, numpy as np\n"
        f"sys.path[:0] = [{ROOT!r}, {os.path.join(ROOT, 'oracle')!r}]\n"
        "import oracle, paper_0910_4711_b200 as vq\n"
        "from paper_0910_4711_b200 import synthetic\n"
        "x = synthetic.make_training('cfg1')[:8192]\n"
        "cb, st = vq.lbg_train(vq.TrainingSet(x), vq.LbgConfig(target_size=64, epsilon=1e-4))\n"
        "ref = oracle.lbg_train(x.astype(np.float64), 64, epsilon=1e-4)\n"
        "assert len(ref.history) > 40, len(ref.history)\n"
        "assert [(h.codebook_size, h.iteration, h.empty_cells) for h in st.history] == "
        "[(s, i, e) for s, i, _, e in ref.history]\n"
        "assert cb.codevectors.tobytes() == ref.codebook.tobytes()\n"
        "print('ok', len(st.history))\n")
    env = dict(os.environ, VQB_HIST_RING="16", VQB_BATCH="4")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.startswith("ok")


# ---------------------------------------------------------------------------
# threads sharing one TrainingSet (ctypes releases the GIL)
# ---------------------------------------------------------------------------

def test_threads_share_a_training_set():
    rng = np.random.default_rng(10)
    x = rng.uniform(0, 255, (200000, 16)).astype(np.float32)
    books = [vq.Codebook(rng.uniform(0, 255, (k, 16))) for k in (64, 256, 1024, 32)]
    ts = vq.TrainingSet(x)
    serial = []
    for b in books:
        t, d = vq.assign_cells(ts, b)
        serial.append((t.cells, d, vq.update_codebook(ts, t, b)[0].codevectors))
    ts2 = vq.TrainingSet(x)  # fresh: the session is created under contention too
    results = [None] * (len(books) * 3)
    errors = []

    def work(i):
        try:
            b = books[i % len(books)]
            t, d = vq.assign_cells(ts2, b)
            results[i] = (t.cells, d, vq.update_codebook(ts2, t, b)[0].codevectors)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(results))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for i, r in enumerate(results):
        c, d, cbk = serial[i % len(books)]
        assert np.array_equal(r[0], c) and r[1] == d and r[2].tobytes() == cbk.tobytes()


# ---------------------------------------------------------------------------
# the candidate pass for float64 rows and every L <= 64
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("dim", [2, 5, 9, 16, 36])
def test_float64_rows_any_dim_fast_path_bit_exact(dim):
    """float64 normals (not float32-exact), N=2^20, K=1024: the FP32 /
    tensor-core candidate pass on the rounded, zero-padded rows with the
    rounding added to the certified band, FP64 re-rank against the float64
    rows -> indices and per-row distances bit-identical to the reference."""
    from paper_0910_4711_b200.core import _Session
    rng = np.random.default_rng(100 + dim)
    x = rng.normal(0, 1, (1 << 20, dim)) * rng.uniform(0.5, 3.0, dim) + rng.uniform(-2, 2, dim)
    cb = x[rng.choice(x.shape[0], 1024, replace=False)] + rng.normal(0, 0.05, (1024, dim))
    s = _Session(None, x)
    info = s.info()
    assert info["fast"] and info["float64_rows"] and info["cdim"] in (16, 32, 64)
    cells, dists, total = s.assign(cb, 0)
    want_c, want_d = oracle.assign_all(x, cb, workers=oracle.max_threads())
    assert np.array_equal(cells, want_c)
    assert dists.tobytes() == want_d.tobytes()
    assert total == oracle.sum_inorder(want_d)


@pytest.mark.parametrize("dim", [3, 5, 36])
def test_float32_rows_any_dim_fast_path_bit_exact(dim):
    from paper_0910_4711_b200.core import _Session
    rng = np.random.default_rng(200 + dim)
    x = rng.uniform(0, 255, (200000, dim)).astype(np.float32)
    cb = rng.uniform(0, 255, (512, dim))
    s = _Session(x, None)
    assert s.info()["fast"] and not s.info()["float64_rows"]
    cells, dists, _ = s.assign(cb, 0)
    want_c, want_d = oracle.assign_all(x.astype(np.float64), cb, workers=oracle.max_threads())
    assert np.array_equal(cells, want_c)
    assert dists.tobytes() == want_d.tobytes()


def test_float64_design_fast_path_matches_reference():
    """A whole float64 design on the candidate pass: schedule, TD and
    codebook bit-identical to the reference (reference-order sums, n <= 2^20)."""
    rng = np.random.default_rng(9)
    x = rng.normal(0, 1, (50000, 7)) * np.array([1.0, 3.0, 0.2, 10.0, 1.0, 0.5, 2.0])
    cb, stats = vq.lbg_train(vq.TrainingSet(x), vq.LbgConfig(target_size=64, epsilon=1e-3))
    ref = oracle.lbg_train(x, 64, epsilon=1e-3, workers=oracle.max_threads())
    assert stats.td_history() == [(s_, i, td) for s_, i, td, _ in ref.history]
    assert cb.codevectors.tobytes() == ref.codebook.tobytes()


# ---------------------------------------------------------------------------
# incremental cell sums (kernels.cu moved_scan / sums_delta / reduce_delta):
# every pass after a level's first updates the running two-word sums by the
# rows that changed cell.  Integer sums are exact, so the design must equal
# the one that sums every row in every pass (VQB_DELTA=0) bit for bit --
# codebook, history (TD, empty cells), per-row distances -- and the oracle.
# Reference: _kernels.update_rows (_kernels.py:39-66), core.py:384-415.
# ---------------------------------------------------------------------------

def _design_both(x, conf, fracs=("0.3", "1.0", "0.0")):
    from paper_0910_4711_b200.core import _Session
    s = _Session(x, None) if x.dtype == np.float32 else _Session(None, x)
    old = {k: os.environ.get(k) for k in ("VQB_DELTA", "VQB_DELTA_FRAC")}
    try:
        os.environ["VQB_DELTA"] = "0"
        ref = s.train(conf)
        outs = []
        for f in fracs:
            os.environ["VQB_DELTA"] = "1"
            os.environ["VQB_DELTA_FRAC"] = f
            outs.append(s.train(conf))
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return ref, outs


def _same_design(a, b):
    ha = [(h.codebook_size, h.iteration, h.td, h.empty_cells) for h in a[1]]
    hb = [(h.codebook_size, h.iteration, h.td, h.empty_cells) for h in b[1]]
    assert ha == hb
    assert np.asarray(a[0]).tobytes() == np.asarray(b[0]).tobytes()
    assert a[3] == b[3]
    assert np.asarray(a[4]).tobytes() == np.asarray(b[4]).tobytes()


@pytest.mark.parametrize("case", ["gmm16", "blocks64", "hetero16", "dim5", "tiny", "f64exact"])
def test_incremental_sums_equal_full_sums(case):
    rng = np.random.default_rng(123)
    if case == "gmm16":
        means = rng.uniform(0, 255, (64, 16))
        x = (means[rng.integers(0, 64, 200001)] + rng.normal(0, 9, (200001, 16))).astype(np.float32)
        conf = vq.LbgConfig(target_size=128, epsilon=1e-4, delta=0.01)
    elif case == "blocks64":   # dimension pieces of the limb tables, integer rows
        x = np.clip(rng.normal(128, 40, (60000, 64)) + rng.normal(0, 25, (60000, 1)), 0, 255)
        x = np.floor(x).astype(np.float32)
        conf = vq.LbgConfig(target_size=256, epsilon=1e-3, delta=0.01)
    elif case == "hetero16":   # low words: columns spanning 1e6 .. 1e-4
        x = _hetero(1 << 17, 16)
        conf = vq.LbgConfig(target_size=32, epsilon=1e-4, delta=0.01)
    elif case == "dim5":       # a dimension outside {16, 32, 64}, ragged row count
        x = rng.normal(0, 1, (33333, 5)).astype(np.float32)
        conf = vq.LbgConfig(target_size=64, epsilon=1e-3, delta=0.01)
    elif case == "tiny":       # fewer rows than one tile, empty cells
        x = rng.integers(0, 4, (37, 3)).astype(np.float32)
        conf = vq.LbgConfig(target_size=16, epsilon=1e-3, delta=0.01)
    else:                      # float64 rows float32 holds exactly
        x = np.floor(rng.normal(0, 300, (40000, 8)))
        conf = vq.LbgConfig(target_size=64, epsilon=1e-3, delta=0.01)
    ref, outs = _design_both(x, conf)
    for out in outs:
        _same_design(ref, out)
    # and the oracle, on the schedule (the codebook where the reference's own sums are exact)
    if case in ("blocks64", "tiny", "f64exact"):
        want = oracle.lbg_train(np.asarray(x, dtype=np.float64), conf.target_size, epsilon=conf.epsilon,
                                delta=conf.delta, workers=oracle.max_threads())
        assert [(h.codebook_size, h.iteration, h.empty_cells) for h in ref[1]] == \
            [(s_, i, e) for s_, i, _, e in want.history]
        assert np.asarray(outs[0][0]).tobytes() == want.codebook.tobytes()


def test_incremental_sums_after_other_calls_on_the_session():
    """assign / update / a second design between designs: the running sums and
    previous cells of a finished design are never reused."""
    from paper_0910_4711_b200.core import _Session
    rng = np.random.default_rng(5)
    x = np.floor(rng.normal(100, 30, (50000, 16))).astype(np.float32)
    s = _Session(x, None)
    conf = vq.LbgConfig(target_size=32, epsilon=1e-3, delta=0.01)
    a = s.train(conf)
    cells, _, _ = s.assign(np.asarray(a[0])[:7].copy(), 0)
    s.update(cells, np.asarray(a[0])[:7].copy())
    b = s.train(vq.LbgConfig(target_size=8, epsilon=1e-3, delta=0.01))
    c = s.train(conf)
    _same_design(a, c)
    want = oracle.lbg_train(x.astype(np.float64), 8, epsilon=1e-3, delta=0.01, workers=oracle.max_threads())
    assert np.asarray(b[0]).tobytes() == want.codebook.tobytes()


# ---------------------------------------------------------------------------
# small codebooks (K < 64): assign_small_kernel at W = 16 (rows staged through
# shared memory) and the difference-form values at W = 32 / 64.  Indices and
# per-row distances must stay the oracle's bit for bit on data built to sit on
# the band's edges.  Reference: _kernels.assign_range (_kernels.py:18-36).
# ---------------------------------------------------------------------------

import functools


@functools.lru_cache(maxsize=1)
def _small_k_cases():
    rng = np.random.default_rng(77)
    out = []
    for dim in (16, 32, 64, 11, 48):
        n = 20011
        # image-like rows: a large mean per row, a small texture on top
        base = rng.integers(20, 236, (n, 1)).astype(np.float64)
        x = np.clip(base + rng.normal(0, 3.0, (n, dim)), 0, 255).round().astype(np.float32)
        for k in (2, 7, 33, 63):
            cb = x[rng.choice(n, k, replace=False)].astype(np.float64)
            cb[k // 2] = cb[0]                     # an exact duplicate: lowest index must win
            cb[-1] = cb[1] + 1e-9                  # a near-duplicate far inside any FP32 band
            out.append((f"blocks_d{dim}_k{k}", x, cb))
        # rows exactly on codevectors (zero distances) and exact two-way ties
        cb = np.zeros((4, dim))
        cb[1, 0], cb[2, 0], cb[3, 1] = 2.0, -2.0, 2.0
        t = rng.integers(-3, 4, (4099, dim)).astype(np.float32) * 0
        t[:, 0] = rng.integers(-3, 4, 4099)
        t[:, 1] = rng.integers(-3, 4, 4099)
        out.append((f"ties_d{dim}", t, cb))
        # a common offset of 1e5 and magnitudes of 1e-3
        out.append((f"offset_d{dim}", (x + 1e5).astype(np.float32), x[:37].astype(np.float64) + 1e5 + 0.25))
        out.append((f"tiny_d{dim}", (x * 1e-5).astype(np.float32), x[:21].astype(np.float64) * 1e-5))
    return out


@pytest.mark.parametrize("i", range(35))  # 5 widths x (4 codebook sizes + ties + offset + tiny)
def test_small_codebook_paths_vs_oracle(i):
    from paper_0910_4711_b200.core import _session_of, _matrix_keep_f32
    name, x, cb = _small_k_cases()[i]
    cells, dists = oracle.assign_all(x.astype(np.float64), cb, workers=oracle.max_threads())
    got_cells, got_d, total = _session_of(_matrix_keep_f32(x)).assign(cb, 0)
    assert np.array_equal(got_cells, cells), name
    assert got_d.tobytes() == dists.tobytes(), name


def test_small_codebook_float64_rows_vs_oracle():
    """float64 rows float32 cannot hold (the candidate rows are rounded copies,
    the winner distance reads the float64 rows) through both small-K paths."""
    from paper_0910_4711_b200.core import _Session
    rng = np.random.default_rng(78)
    for dim, k in ((16, 9), (64, 31), (5, 40)):
        x = rng.normal(100.0, 30.0, (30011, dim)) + rng.normal(0, 1e-7, (30011, dim))
        cb = x[rng.choice(30011, k, replace=False)] + 0.125
        cells, dists = oracle.assign_all(x, cb, workers=oracle.max_threads())
        got_cells, got_d, _ = _Session(None, x).assign(cb, 0)
        assert np.array_equal(got_cells, cells), (dim, k)
        assert got_d.tobytes() == dists.tobytes(), (dim, k)
