"""Parity of the B200 path (libvqb200.so through the drop-in API) against the
reference's golden vectors and the CPU oracle.  GPU only."""

import hashlib
import os

import numpy as np
import pytest

import cases
import oracle
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

vq = pytest.importorskip("paper_0910_4711_b200")


def _golden(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{name} golden not generated")
    return np.load(path)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    from paper_0910_4711_b200 import _lib
    if _lib.device_count() < 1:
        pytest.fail("GPU tests need a CUDA device")


# ---------------------------------------------------------------------------
# allocation: indices and per-row FP64 distances bit-exact
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("i", range(len(cases.assign_cases())))
def test_assign_matches_reference(golden_small, i):
    case = cases.assign_cases()[i]
    metric = ["squared_euclidean", "euclidean"][case["metric"]]
    table, total = vq.assign_cells(case["x"], vq.Codebook(case["cb"]), metric=metric)
    assert table.cells.dtype == np.int64
    assert np.array_equal(table.cells, golden_small[f"assign{i}_cells"])
    # chunks <= 2^20 rows: the total is accumulated in input order, as the reference
    assert total == float(golden_small[f"assign{i}_total"])


@pytest.mark.parametrize("i", range(len(cases.assign_cases())))
def test_assign_dists_bit_exact(golden_small, i):
    case = cases.assign_cases()[i]
    from paper_0910_4711_b200.core import _session_of, _matrix_keep_f32
    _, dists, _ = _session_of(_matrix_keep_f32(case["x"])).assign(case["cb"], case["metric"])
    assert dists.tobytes() == golden_small[f"assign{i}_dists"].tobytes()


def test_assign_float32_input_uses_fast_path_and_matches():
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 255, (50000, 16)).astype(np.float32)
    cb = rng.uniform(0, 255, (1024, 16))
    cells, dists = oracle.assign_all(x.astype(np.float64), cb, workers=8)
    table, _ = vq.assign_cells(x, vq.Codebook(cb))
    assert np.array_equal(table.cells, cells)


@pytest.mark.parametrize("dim,k", [(16, 2), (16, 64), (16, 128), (16, 4096), (32, 300), (32, 128),
                                   (64, 64), (64, 512), (64, 1)])
def test_assign_shapes_vs_oracle(dim, k):
    rng = np.random.default_rng(dim * 1000 + k)
    x = rng.integers(0, 256, (20000, dim)).astype(np.float32)
    cb = x[rng.choice(20000, k, replace=False)].astype(np.float64) + 0.5
    cells, _ = oracle.assign_all(x.astype(np.float64), cb, workers=8)
    table, _ = vq.assign_cells(x, vq.Codebook(cb))
    assert np.array_equal(table.cells, cells)


def _adversarial_cases():
    rng = np.random.default_rng(77)
    out = []
    # large common offset: distances tiny against the norms (cancellation in
    # |x|^2 - 2xc + |c|^2); the certified band must queue, never mis-rank
    x = (1.0e5 + rng.normal(0, 1, (12345, 16))).astype(np.float32)
    out.append(("offset-L16", x, x[rng.choice(len(x), 1024, replace=False)].astype(np.float64) + 0.25))
    # tiny magnitudes, L=32
    x = rng.uniform(0, 1e-3, (9001, 32)).astype(np.float32)
    out.append(("tiny-L32", x, rng.uniform(0, 1e-3, (256, 32))))
    # negative values, every codevector twice (exact ties), L=64
    x = rng.integers(-128, 128, (7777, 64)).astype(np.float32)
    cb = rng.integers(-128, 128, (32, 64)).astype(np.float64)
    out.append(("dup-neg-L64", x, np.repeat(cb, 2, axis=0)))
    # rows sitting exactly on codevectors (zero distances), L=16, K=512
    cb = rng.integers(0, 256, (512, 16)).astype(np.float64)
    x = cb[rng.integers(0, 512, 10000)].astype(np.float32)
    out.append(("on-codevector-L16", x, cb))
    # dimensions off the tensor-core set
    for dim, k in ((3, 100), (48, 200), (100, 64), (128, 256)):
        x = rng.integers(0, 256, (5003, dim)).astype(np.float32)
        out.append((f"dim{dim}", x, x[rng.choice(5003, k, replace=False)].astype(np.float64) + 0.5))
    return out


@pytest.mark.parametrize("i", range(8))
def test_assign_adversarial_vs_oracle(i):
    """Offsets, tiny magnitudes, negative duplicates, zero distances, ragged
    row counts and dimensions outside 16/32/64: indices and per-row distances
    stay the oracle's bit for bit."""
    name, x, cb = _adversarial_cases()[i]
    cells, dists = oracle.assign_all(x.astype(np.float64), cb, workers=8)
    from paper_0910_4711_b200.core import _session_of, _matrix_keep_f32
    table, _ = vq.assign_cells(x, vq.Codebook(cb))
    assert np.array_equal(table.cells, cells), name
    _, got, _ = _session_of(_matrix_keep_f32(x)).assign(cb, 0)
    assert got.tobytes() == dists.tobytes(), name
    stream = vq.encode(x, vq.Codebook(cb))
    assert np.array_equal(stream.indices, cells.astype(np.uint32)), name


def test_first_split_tie_density_exact():
    """K=2 additive split of a GMM centroid: the tie-densest point of the whole
    design.  Indices must still be bit-exact."""
    from paper_0910_4711_b200 import synthetic
    x = synthetic.make_training("cfg2", n=1 << 18)
    x64 = x.astype(np.float64)
    c = oracle.column_sums(x64) / x.shape[0]
    cb = oracle.split_rows(c.reshape(1, -1), 0.01)
    cells, _ = oracle.assign_all(x64, cb, workers=8)
    table, _ = vq.assign_cells(x, vq.Codebook(cb))
    assert np.array_equal(table.cells, cells)


# ---------------------------------------------------------------------------
# update
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("i", range(len(cases.update_cases())))
def test_update_matches_reference(golden_small, i):
    case = cases.update_cases()[i]
    ts = vq.TrainingSet(case["x"])
    table = vq.CellTable(case["cells"], case["cb"].shape[0])
    cb, empty = vq.update_codebook(ts, table, vq.Codebook(case["cb"]))
    want = golden_small[f"update{i}_cb"]
    assert empty == int(np.count_nonzero(golden_small[f"update{i}_counts"] == 0))
    if i == 5:
        # tiny and large magnitudes in one huge cell: the reference's sequential
        # sum rounds, the device's exact fixed-point sum does not -> ulps apart
        np.testing.assert_allclose(cb.codevectors, want, rtol=1e-13, atol=1e-13)
    else:
        assert cb.codevectors.tobytes() == want.tobytes()


# ---------------------------------------------------------------------------
# full designs
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("i", range(len(cases.design_cases())))
def test_design_matches_reference(golden_small, i):
    case = cases.design_cases()[i]
    cfg = vq.LbgConfig(**case["config"])
    cb, stats = vq.parallel_lbg_train(vq.TrainingSet(case["x"]), cfg)
    hist = np.array([(h.codebook_size, h.iteration, h.td, h.empty_cells) for h in stats.history],
                    dtype=np.float64).reshape(-1, 4)
    want_hist = golden_small[f"design{i}_hist"]
    assert hist.shape == want_hist.shape
    assert np.array_equal(hist[:, [0, 1, 3]], want_hist[:, [0, 1, 3]])
    np.testing.assert_allclose(hist[:, 2], want_hist[:, 2], rtol=1e-12, atol=0)
    np.testing.assert_allclose(cb.codevectors, golden_small[f"design{i}_cb"], rtol=1e-12, atol=1e-12)
    assert len(stats.warnings) == int(golden_small[f"design{i}_nwarn"])
    np.testing.assert_allclose(stats.per_worker, golden_small[f"design{i}_per_worker"], rtol=1e-12)


@pytest.mark.parametrize("dim,k,offset", [(16, 64, 1000.0), (32, 32, -300.0), (64, 16, 0.0)])
def test_design_offset_integer_data_vs_oracle(dim, k, offset):
    """Whole designs on integer-valued rows far from the origin (and
    negative): every FP64 cell sum is exact on both sides, so the codebooks
    are bit-identical and the schedules match pass for pass."""
    rng = np.random.default_rng(dim + k)
    x = (offset + rng.integers(-50, 51, (20011, dim))).astype(np.float32)
    want = oracle.lbg_train(x.astype(np.float64), k, epsilon=1e-3, delta=0.01, workers=8)
    cb, stats = vq.lbg_train(vq.TrainingSet(x), vq.LbgConfig(target_size=k, epsilon=1e-3, delta=0.01))
    hist = np.array([(h.codebook_size, h.iteration, h.td, h.empty_cells) for h in stats.history])
    ref = np.array(want.history, dtype=np.float64)
    assert np.array_equal(hist[:, [0, 1, 3]], ref[:, [0, 1, 3]])
    np.testing.assert_allclose(hist[:, 2], ref[:, 2], rtol=2 * x.shape[0] * 2.0 ** -53)
    assert cb.codevectors.tobytes() == np.ascontiguousarray(want.codebook).tobytes()


def test_trace_kat_exact():
    trace = vq.TrainingSet(np.array([[0.0, 0.0], [0.0, 1.0], [4.0, 0.0], [4.0, 1.0]]))
    cb, stats = vq.lbg_train(trace, vq.LbgConfig(target_size=2, epsilon=1e-3, delta=0.5))
    assert cb.codevectors.tolist() == [[4.0, 0.5], [0.0, 0.5]]
    assert stats.total == 1.0
    assert stats.td_history() == [(2, 1, 11.0), (2, 2, 1.0), (2, 3, 1.0)]
    assert stats.mean == 0.25


def _design_check(cfg_name, g, x, rtol_td=None):
    # The reference sums TD left to right, the device in a fixed tile tree:
    # both are within n*u of the exact sum (u = 2^-53), so they agree to
    # ~2nu -- far inside the north star's 1e-4.
    if rtol_td is None:
        rtol_td = max(1e-12, 2.0 * x.shape[0] * 2.0 ** -53)
    from paper_0910_4711_b200 import synthetic
    spec = synthetic.WORKLOADS[cfg_name]
    assert hashlib.sha256(x.tobytes()).hexdigest() == g["x_sha256"].item().decode()
    conf = vq.LbgConfig(target_size=spec.target_size, epsilon=spec.epsilon, delta=spec.delta)
    cb, stats = vq.lbg_train(vq.TrainingSet(x), conf)
    hist = np.array([(h.codebook_size, h.iteration, h.td, h.empty_cells) for h in stats.history])
    want = g["hist"]
    # iteration count and per-level schedule must match exactly
    assert hist.shape == want.shape, (hist.shape, want.shape)
    assert np.array_equal(hist[:, [0, 1, 3]], want[:, [0, 1, 3]])
    np.testing.assert_allclose(hist[:, 2], want[:, 2], rtol=rtol_td)
    assert abs(stats.total - float(g["total"])) <= 1e-4 * float(g["total"])
    np.testing.assert_allclose(cb.codevectors, g["cb"], rtol=1e-5)
    return cb, stats


def test_cfg1_full_design_vs_reference():
    from paper_0910_4711_b200 import synthetic
    g = _golden("cfg1_design")
    cb, _ = _design_check("cfg1", g, synthetic.make_training("cfg1"))
    # 8-bit pixels: every FP64 sum is exact, so the codebook is bit-identical
    assert cb.codevectors.tobytes() == g["cb"].tobytes()


def test_cfg2_full_design_vs_reference():
    from paper_0910_4711_b200 import synthetic
    g = _golden("cfg2_design")
    _design_check("cfg2", g, synthetic.make_training("cfg2"))


def test_cfg3_full_design_vs_reference():
    """L=64 image blocks (BASELINE configs[2]): 8-bit pixels, so the whole
    design is bit-identical to the reference's."""
    from paper_0910_4711_b200 import synthetic
    g = _golden("cfg3_design")
    cb, _ = _design_check("cfg3", g, synthetic.make_training("cfg3"))
    assert cb.codevectors.tobytes() == g["cb"].tobytes()


def test_cfg4_full_design_vs_reference():
    """N=2^24, K=4096 (BASELINE configs[3]) on one device."""
    from paper_0910_4711_b200 import synthetic
    g = _golden("cfg4_design")
    _design_check("cfg4", g, synthetic.make_training("cfg4"))


def test_cfg5_encode_vs_reference():
    """2^26 queries against the fixed K=1024 codebook (BASELINE configs[4]):
    indices bit-identical to the reference's encode, distortion to 1e-12."""
    from paper_0910_4711_b200 import synthetic
    g = _golden("cfg5_encode")
    cb, q = synthetic.make_encode_case()
    assert hashlib.sha256(q.tobytes()).hexdigest() == g["q_sha256"].item().decode()
    stream = vq.encode(q, vq.Codebook(cb.astype(np.float64)))
    assert stream.indices.dtype == np.uint32
    assert np.array_equal(stream.indices[:65536], g["head"])
    assert np.array_equal(np.bincount(stream.indices, minlength=1024), g["bincount"])
    assert hashlib.sha256(stream.indices.tobytes()).hexdigest() == g["idx_sha256"].item().decode()
    del stream
    _, total = vq.assign_cells(q, vq.Codebook(cb.astype(np.float64)))
    assert abs(total - float(g["total"])) <= 1e-12 * float(g["total"])


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_teacher_forced_counts(cfg):
    """Every recorded codebook of the reference run, fed to the device, gives
    the reference's cell counts exactly."""
    from paper_0910_4711_b200 import synthetic
    g = _golden(f"{cfg}_design")
    x = synthetic.make_training(cfg)
    ts = vq.TrainingSet(x)
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
    assert checked > 10
    # the reference's final codebook too (its last pass converged on it)
    table, _ = vq.assign_cells(ts, vq.Codebook(g["cb"]))
    assert np.array_equal(np.bincount(table.cells, minlength=g["cb"].shape[0]),
                          counts[offs[-2]:offs[-1]])


# ---------------------------------------------------------------------------
# encode
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("i", range(len(cases.encode_cases())))
def test_encode_matches_reference(golden_small, i):
    case = cases.encode_cases()[i]
    stream = vq.encode(case["x"], vq.Codebook(case["cb"]), workers=case["workers"])
    assert stream.indices.dtype == np.uint32
    assert np.array_equal(stream.indices, golden_small[f"encode{i}_idx"])


def test_encode_float32_pipeline_vs_oracle():
    from paper_0910_4711_b200 import synthetic
    cb, q = synthetic.make_encode_case(n=(1 << 22) + 12345)  # > one pipeline chunk
    stream = vq.encode(q, vq.Codebook(cb.astype(np.float64)))
    sub = slice(0, 200000)
    cells, _ = oracle.assign_all(q[sub].astype(np.float64), cb.astype(np.float64), workers=8)
    assert np.array_equal(stream.indices[sub], cells.astype(np.uint32))
    tail = slice(q.shape[0] - 50000, q.shape[0])
    cells, _ = oracle.assign_all(q[tail].astype(np.float64), cb.astype(np.float64), workers=8)
    assert np.array_equal(stream.indices[tail], cells.astype(np.uint32))


def test_empty_encode_and_errors():
    cb = vq.Codebook(np.zeros((2, 3)))
    assert len(vq.encode(np.empty((0, 3)), cb)) == 0
    with pytest.raises(vq.UsageError):
        vq.assign_cells(np.empty((0, 3)), cb)
    with pytest.raises(vq.UsageError, match="dimension"):
        vq.encode(np.zeros((4, 2)), cb)


def test_determinism_repeat_runs():
    from paper_0910_4711_b200 import synthetic
    x = synthetic.make_training("cfg2", n=1 << 16)
    cfg = vq.LbgConfig(target_size=64, epsilon=1e-4, delta=0.01)
    cb1, s1 = vq.lbg_train(vq.TrainingSet(x), cfg)
    cb2, s2 = vq.lbg_train(vq.TrainingSet(x.copy()), cfg)
    assert cb1.codevectors.tobytes() == cb2.codevectors.tobytes()
    assert s1.td_history() == s2.td_history()


# ---------------------------------------------------------------------------
# kernel surface (drop-in for vqkit._kernels) against the reference's outputs
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("i", range(len(cases.assign_cases())))
def test_kernel_surface_assign_range(golden_small, i):
    from paper_0910_4711_b200 import kernels
    case = cases.assign_cases()[i]
    m = case["x"].shape[0]
    cells = np.full(m, -7, dtype=np.int64)
    dists = np.full(m, -1.0)
    lo, hi = m // 3, m
    kernels.assign_range(case["x"], case["cb"], 0, lo, case["metric"], cells, dists)
    kernels.assign_range(case["x"], case["cb"], lo, hi, case["metric"], cells, dists)
    assert np.array_equal(cells, golden_small[f"assign{i}_cells"])
    assert dists.tobytes() == golden_small[f"assign{i}_dists"].tobytes()
    assert kernels.sum_inorder(dists) == float(golden_small[f"assign{i}_total"])


@pytest.mark.parametrize("i", range(len(cases.update_cases())))
def test_kernel_surface_update_rows_round_robin(golden_small, i):
    """update_rows over a (worker, stride) decomposition, as parallel_update
    drives it (parallel.py:144-154), equals the reference's single-worker run."""
    from paper_0910_4711_b200 import kernels
    case = cases.update_cases()[i]
    cb = case["cb"]
    out = np.full_like(cb, np.nan)
    counts = np.full(cb.shape[0], -1, dtype=np.int64)
    for w in range(3):
        kernels.update_rows(case["x"], case["cells"], cb, w, 3, out, counts)
    assert np.array_equal(counts, golden_small[f"update{i}_counts"])
    want = golden_small[f"update{i}_cb"]
    if i == 5:
        np.testing.assert_allclose(out, want, rtol=1e-13, atol=1e-13)
    else:
        assert out.tobytes() == want.tobytes()


def test_kernel_surface_small_helpers():
    from paper_0910_4711_b200 import kernels
    rng = np.random.default_rng(3)
    x = rng.normal(size=(1000, 5))
    assert kernels.column_sums(x).tobytes() == oracle.column_sums(x).tobytes()
    assert kernels.sum_inorder(x[:, 0]) == oracle.sum_inorder(x[:, 0])
    assert kernels.pair_distance(x[0], x[1], 1) == oracle.pair_distance(x[0], x[1], 1)
    assert kernels.pair_distance(x[0], x[1], 0) == oracle.pair_distance(x[0], x[1], 0)


# ---------------------------------------------------------------------------
# host-buffer entry points (transfer engine: pinned and pageable sources)
# ---------------------------------------------------------------------------

def _pinned_copy(a):
    torch = pytest.importorskip("torch")
    t = torch.from_numpy(a).pin_memory()
    return t, t.numpy()


@pytest.mark.parametrize("pinned", [False, True])
def test_lloyd_step_f32_host_buffers(pinned):
    import ctypes
    from paper_0910_4711_b200 import _lib, synthetic
    g = _golden("cfg2_design")
    x = synthetic.make_training("cfg2", n=(1 << 18) + 777)
    keep = None
    if pinned:
        keep, x = _pinned_copy(x)
    last = max(int(k[4:-3]) for k in g.files if k.startswith("pass") and k.endswith("_cb"))
    cb = np.ascontiguousarray(g[f"pass{last}_cb"])  # a K=64 codebook of the reference's run
    k = cb.shape[0]
    new = np.empty_like(cb)
    cells = np.empty(x.shape[0], dtype=np.int64)
    td, empty = ctypes.c_double(), ctypes.c_int64()
    _lib.check(_lib.lib().vqb_lloyd_step_f32(_lib.ptr(x), x.shape[0], 16, _lib.ptr(cb), k, 0,
                                             _lib.ptr(new), _lib.ptr(cells), ctypes.byref(td),
                                             ctypes.byref(empty)))
    x64 = x.astype(np.float64)
    want_cells, dists = oracle.assign_all(x64, cb, workers=8)
    assert np.array_equal(cells, want_cells)
    want_cb, counts = oracle.update_all(x64, want_cells, cb, workers=8)
    np.testing.assert_allclose(new, want_cb, rtol=1e-13, atol=0)
    assert empty.value == int(np.count_nonzero(counts == 0))
    assert abs(td.value - oracle.sum_inorder(dists)) <= 1e-12 * td.value
    del keep


@pytest.mark.parametrize("pinned", [False, True])
def test_encode_f32_host_buffers_and_total(pinned):
    import ctypes
    from paper_0910_4711_b200 import _lib, synthetic
    cb32, q = synthetic.make_encode_case(n=(1 << 22) * 2 + 4097)  # 3 pipeline chunks
    keep = None
    if pinned:
        keep, q = _pinned_copy(q)
    cb = cb32.astype(np.float64)
    idx = np.empty(q.shape[0], dtype=np.uint32)
    total = ctypes.c_double()
    _lib.check(_lib.lib().vqb_encode_f32(_lib.ptr(q), q.shape[0], 16, _lib.ptr(cb), cb.shape[0], 0,
                                         _lib.ptr(idx), ctypes.byref(total)))
    for sl in (slice(0, 100000), slice((1 << 22) - 5000, (1 << 22) + 5000),
               slice(q.shape[0] - 60000, q.shape[0])):
        cells, _ = oracle.assign_all(q[sl].astype(np.float64), cb, workers=8)
        assert np.array_equal(idx[sl], cells.astype(np.uint32))
    _, want_total = vq.assign_cells(q, vq.Codebook(cb))
    assert abs(total.value - want_total) <= 1e-10 * want_total
    del keep


# ---------------------------------------------------------------------------
# tensor-core candidate pass: raw accumulators vs a float64 emulation
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("dim,k", [(16, 1024), (32, 256), (64, 512)])
def test_tc_accumulators_vs_float64_emulation(dim, k):
    """The tcgen05 MMA chain (fp16 hi/lo operands, fp32 TMEM accumulation)
    against the exact value of the same operands: the error stays inside the
    certification band's accumulation term (2 x 2^-22 of the magnitude sum
    per MMA), with a 2x margin."""
    import tc_emulation as te
    from paper_0910_4711_b200 import _lib
    from paper_0910_4711_b200.core import _Session
    rng = np.random.default_rng(dim + k)
    x = rng.normal(100, 40, (1000, dim)).astype(np.float32)
    cb = rng.normal(100, 40, (k, dim))
    s = _Session(x, None)
    dump = np.empty((128, k), dtype=np.float32)
    sc = np.zeros(5, dtype=np.int32)
    _lib.check(_lib.lib().vqb_debug_tc_tile(s.handle, _lib.ptr(cb), k, _lib.ptr(dump), _lib.ptr(sc)))
    assert sc[3] == 1 and sc[4] == 0  # TC pass configured, codebook representable
    d, mag, v = te.expected_accumulators(x[:128], te.session_mu(x), cb, int(sc[0]), int(sc[1]), int(sc[2]))
    rel = np.abs(dump.astype(np.float64) - d) / mag
    n_mma = 3 * dim // 16 + 1
    assert rel.max() <= 0.5 * 2 * n_mma * 2.0 ** -22, rel.max()
    assert np.array_equal(np.argmin(dump, 1), np.argmin(v, 1))


# ---------------------------------------------------------------------------
# split_codebook on the device (core.py:277-289)
# ---------------------------------------------------------------------------

def test_split_codebook_known_answers_and_oracle():
    # the reference's split KATs (pkg/tests/test_core.py split tests)
    assert vq.split_codebook(vq.Codebook([(2.0, 0.5)]), 0.5).codevectors.tolist() == [[2.5, 1.0], [1.5, 0.0]]
    got = vq.split_codebook(vq.Codebook([(0.0, 0.0), (4.0, 4.0)]), 0.01).codevectors.tolist()
    assert got == [[0.01, 0.01], [-0.01, -0.01], [4.01, 4.01], [3.99, 3.99]]
    rows = np.random.default_rng(5).normal(0, 100, (37, 13))
    for delta in (0.01, 0.005, 1e-9):
        out = vq.split_codebook(vq.Codebook(rows), delta).codevectors
        assert out.tobytes() == oracle.split_rows(rows, delta).tobytes()
    with pytest.raises(vq.ConfigError):
        vq.split_codebook(vq.Codebook(rows), 0.0)


def _tc_edge_operands(kind, dim, k, rng):
    """Operand sets aimed at the accumulation term of the certification band."""
    if kind == "cancel":      # a large common mean, a small spread: ||c||^2 and 2 y.c cancel to ~1e-4 of their size
        base = rng.normal(0, 1, dim) * 200 + 500
        x = (base + rng.normal(0, 0.5, (1000, dim))).astype(np.float32)
        cb = base + rng.normal(0, 0.5, (k, dim))
        x[::2] += 300                               # rows far from the session mean: |y| large, distances small
        cb[::2] += 300
    elif kind == "signs":     # alternating signs: every partial sum of an MMA cancels
        sgn = np.where(np.arange(dim) % 2 == 0, 1.0, -1.0)
        x = (rng.uniform(200, 255, (1000, dim)) * sgn).astype(np.float32)
        cb = rng.uniform(200, 255, (k, dim)) * sgn * np.where(rng.random((k, 1)) < 0.5, 1.0, -1.0)
    elif kind == "ones":      # mantissas of all ones: the fp16 hi/lo split rounds up and the low word is negative
        m = (2.0 ** 24 - 1) / 2.0 ** 24
        x = (m * 2.0 ** rng.integers(0, 8, (1000, dim))).astype(np.float32)
        cb = m * 2.0 ** rng.integers(0, 8, (k, dim)).astype(np.float64) + 2.0 ** -20
    else:                     # "range": dimensions and codevectors over 4 decades
        scale = 10.0 ** rng.uniform(-2, 2, dim)
        x = (rng.normal(0, 1, (1000, dim)) * scale).astype(np.float32)
        cb = rng.normal(0, 1, (k, dim)) * scale * 10.0 ** rng.uniform(-1, 0, (k, 1))
    return x, cb


@pytest.mark.parametrize("kind", ["cancel", "signs", "ones", "range"])
@pytest.mark.parametrize("dim,k", [(16, 4096), (16, 256), (32, 768), (64, 512), (64, 2048)])
def test_tc_accumulators_band_edge_operands(kind, dim, k):
    """The emulation test on operands built against the accumulation bound
    (VERDICT r1 weak #2): heavy cancellation, alternating signs, all-ones
    mantissas, four decades of range; codebooks resident in shared memory and
    streaming through the ring (K = 4096 at L = 16, 2048 at L = 64).  The measured error must stay
    inside HALF of the band's accumulation term, and the accumulators' argmin
    must be the exact operands' argmin wherever the exact gap exceeds it."""
    import tc_emulation as te
    from paper_0910_4711_b200 import _lib
    from paper_0910_4711_b200.core import _Session
    rng = np.random.default_rng(sum(map(ord, kind)) * 1000003 + dim * 8191 + k)
    x, cb = _tc_edge_operands(kind, dim, k, rng)
    s = _Session(x, None)
    dump = np.empty((128, k), dtype=np.float32)
    sc = np.zeros(5, dtype=np.int32)
    _lib.check(_lib.lib().vqb_debug_tc_tile(s.handle, _lib.ptr(cb), k, _lib.ptr(dump), _lib.ptr(sc)))
    if not (sc[3] == 1 and sc[4] == 0):
        pytest.skip("operands outside the fp16 range of the TC pass (the FP32 kernel takes them)")
    d, mag, v = te.expected_accumulators(x[:128], te.session_mu(x), cb, int(sc[0]), int(sc[1]), int(sc[2]))
    err = np.abs(dump.astype(np.float64) - d)
    n_mma = 3 * dim // 16 + 1
    budget = 2 * n_mma * 2.0 ** -22 * mag
    assert (err <= 0.5 * budget).all(), float((err / budget).max())
    # wherever the exact top-2 gap is wider than the measured error allows, the winner agrees
    order = np.sort(d, axis=1)
    clear = (order[:, 1] - order[:, 0]) > 2 * budget.max(axis=1)
    assert np.array_equal(np.argmin(dump, 1)[clear], np.argmin(d, 1)[clear])
