"""Device kernels for the formats either side of the LBG path (imaging.cu via
include/vqb200.h): block vectoriser, raster, decode, fused decode-to-pixels,
reconstruction distortion and the pixel-fed training session -- bit-exact
against the reference's outputs (tests/golden/storage.npz) and the oracle.
GPU only."""

import ctypes
import os

import numpy as np
import pytest

import cases
import oracle
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

vq = pytest.importorskip("paper_0910_4711_b200")
from paper_0910_4711_b200 import _lib, storage, synthetic  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if _lib.device_count() < 1:
        pytest.fail("GPU tests need a CUDA device")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLDEN, "storage.npz"))


@pytest.mark.parametrize("i", range(len(cases.image_cases())))
def test_pixels_to_blocks_bit_exact(gold, i):
    px, b = cases.image_cases()[i]
    vec, grid = vq.pixels_to_blocks(px, b)
    assert vec.dtype == np.float64
    assert vec.tobytes() == gold[f"img{i}_blocks"].tobytes()
    assert [grid.width, grid.height, grid.block, grid.count, grid.k] == gold[f"img{i}_grid"].tolist()
    v32, _ = storage.pixels_to_blocks(px, b, dtype=np.float32)
    assert np.array_equal(v32.astype(np.float64), vec)


@pytest.mark.parametrize("i", range(len(cases.image_cases())))
def test_blocks_to_image_bytes_match_reference(gold, i):
    px, b = cases.image_cases()[i]
    vec = gold[f"img{i}_blocks"]
    grid = storage.BlockGrid(width=px.shape[1], height=px.shape[0], block=b)
    assert vq.blocks_to_image(vec, grid) == gold[f"img{i}_pgm_identity"].tobytes()
    pert = cases.raster_vectors(vec, 100 + i)
    assert vq.blocks_to_image(pert, grid) == gold[f"img{i}_pgm"].tobytes()


def test_blocks_to_image_clamps_and_rounds_half_up():
    # test_storage.py:257-263 of the reference
    out = vq.parse_pgm(vq.blocks_to_image(np.array([[-3.2], [991.0]]), storage.BlockGrid(2, 1, 1)))
    assert out.tolist() == [[0, 255]]
    out = vq.parse_pgm(vq.blocks_to_image(np.array([[0.5], [1.49], [2.5]]), storage.BlockGrid(3, 1, 1)))
    assert out.tolist() == [[1, 1, 3]]
    with pytest.raises(vq.UsageError, match="expected 4 vectors"):
        vq.blocks_to_image(np.zeros((3, 4)), storage.BlockGrid(width=4, height=4, block=2))


def test_image_stack_is_the_concatenation():
    rng = np.random.default_rng(8)
    stack = rng.integers(0, 256, (5, 37, 53), dtype=np.uint8)
    vec, grid = vq.pixels_to_blocks(stack, 8)
    want = np.concatenate([oracle.pixels_to_blocks(im, 8) for im in stack])
    assert vec.tobytes() == want.tobytes()
    back = storage.blocks_to_pixels(vec, grid, images=5)
    assert np.array_equal(back, stack)


@pytest.mark.parametrize("i", range(len(cases.decode_cases())))
def test_decode_bit_exact(gold, i):
    c = cases.decode_cases()[i]
    cb = vq.Codebook(c["cb"])
    rows = vq.decode(vq.EncodedStream(cb.size, cb.k, c["idx"]), cb)
    assert rows.dtype == np.float64 and rows.tobytes() == gold[f"dec{i}_rows"].tobytes()


def test_decode_rejects_out_of_range_index_on_device():
    cb = np.arange(8.0).reshape(4, 2)
    idx = np.array([0, 3, 4, 1], dtype=np.uint32)
    out = np.empty((4, 2))
    rc = _lib.lib().vqb_decode(_lib.ptr(idx), 4, _lib.ptr(cb), 4, 2, 0, _lib.ptr(out))
    assert rc == _lib.VQB_FORMAT
    with pytest.raises(vq.FormatError):
        _lib.check(rc)


def test_decode_empty_and_mismatch():
    cb = vq.Codebook(np.ones((4, 3)))
    assert vq.decode(vq.EncodedStream(4, 3, np.empty(0, dtype=np.uint32)), cb).shape == (0, 3)
    with pytest.raises(vq.UsageError, match="encoded against"):
        vq.decode(vq.EncodedStream(8, 3, [1]), cb)
    with pytest.raises(vq.UsageError, match="dimension"):
        vq.decode(vq.EncodedStream(4, 2, [1]), cb)


@pytest.mark.parametrize("b", [2, 3, 4, 8, 16])
@pytest.mark.parametrize("w", [95, 100, 96])  # band path / 4-pixel path / 16-pixel path
def test_decode_pixels_equals_raster_of_decode(b, w):
    rng = np.random.default_rng(b)
    px = rng.integers(0, 256, (61, w), dtype=np.uint8)
    vec, grid = vq.pixels_to_blocks(px, b)
    cb = vq.Codebook(rng.normal(128, 90, (32, b * b)))
    stream = vq.encode(vec, cb)
    fused = storage.decode_image(stream, cb, grid)
    assert fused == vq.blocks_to_image(vq.decode(stream, cb), grid)
    want = oracle.blocks_to_pixels(oracle.decode(oracle.encode(vec, cb.codevectors), cb.codevectors),
                                   61, w, b)
    assert vq.parse_pgm(fused).tobytes() == want.tobytes()


def test_decode_pixels_rejects_corrupt_indices():
    cb = np.ones((4, 4))
    idx = np.array([0, 1, 2, 7], dtype=np.uint32)
    out = np.empty((4, 4), dtype=np.uint8)
    rc = _lib.lib().vqb_decode_pixels(_lib.ptr(idx), 1, 4, 4, 2, _lib.ptr(cb), 4, 0, _lib.ptr(out))
    assert rc == _lib.VQB_FORMAT


@pytest.mark.parametrize("i", range(len(cases.distortion_cases())))
def test_reconstruction_distortion_bit_exact(gold, i):
    c = cases.distortion_cases()[i]
    total, mean = vq.reconstruction_distortion(c["a"], c["b"], c["metric"])
    assert total == float(gold[f"dist{i}_total"])
    assert mean == float(gold[f"dist{i}_mean"])


def test_reconstruction_distortion_errors():
    with pytest.raises(vq.UsageError, match="length mismatch"):
        vq.reconstruction_distortion(np.ones((3, 2)), np.ones((4, 2)))
    with pytest.raises(vq.UsageError, match="dimension mismatch"):
        vq.reconstruction_distortion(np.ones((3, 2)), np.ones((3, 4)))
    assert vq.reconstruction_distortion(np.empty((0, 2)), np.empty((0, 2))) == (0.0, 0.0)


def test_encode_decode_round_trip_large():
    """Size-independent property at 2^22 rows (cfg5 generator): the distortion
    of decode(encode(x)) equals encode's own per-row minimum distances, the
    indices match the oracle, and the tree-order total is within 1e-13 of the
    in-order sum."""
    cb32, x = synthetic.make_encode_case(1 << 22)
    cb = vq.Codebook(cb32)
    stream = vq.encode(x, cb)
    rec = vq.decode(stream, cb)
    total, _ = vq.reconstruction_distortion(x, rec)
    _, assign_total = vq.assign_cells(x, cb)
    assert abs(total - assign_total) <= 1e-13 * assign_total
    sample = slice(0, 1 << 16)
    cells, dists = oracle.assign_all(x[sample].astype(np.float64), cb.codevectors)
    assert np.array_equal(stream.indices[sample], cells.astype(np.uint32))
    assert np.array_equal(rec[sample], cb.codevectors[cells])


def test_image_training_set_design_matches_host_vectors():
    px = synthetic.make_training_pixels("cfg1")
    ts, grid = storage.image_training_set(px, 4)
    vec, _ = vq.pixels_to_blocks(px, 4)
    assert ts.vectors.tobytes() == vec.tobytes()
    cfg = vq.LbgConfig(target_size=64, epsilon=1e-3, delta=0.01)
    cb1, st1 = vq.lbg_train(ts, cfg)
    cb2, st2 = vq.lbg_train(vq.TrainingSet(vec), cfg)
    assert cb1.codevectors.tobytes() == cb2.codevectors.tobytes()
    assert [(h.codebook_size, h.iteration, h.td) for h in st1.history] == \
        [(h.codebook_size, h.iteration, h.td) for h in st2.history]


def test_open_pixels_validates():
    h = ctypes.c_void_p()
    px = np.zeros((4, 4), dtype=np.uint8)
    assert _lib.lib().vqb_open_pixels(_lib.ptr(px), 1, 4, 4, 0, 0, ctypes.byref(h)) == _lib.VQB_USAGE
    assert _lib.lib().vqb_open_pixels(_lib.ptr(px), 1, 0, 4, 2, 0, ctypes.byref(h)) == _lib.VQB_USAGE
