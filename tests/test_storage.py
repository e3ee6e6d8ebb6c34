"""Formats either side of the LBG path, CPU side:

* the oracle's restatements of pixels_to_blocks / blocks_to_image / decode /
  reconstruction_distortion pinned against the reference's outputs
  (tests/golden/storage.npz, made by make_storage_golden.py);
* the host file formats (VQCB / VQEN byte images, PGM parsing) against the
  same goldens and the reference's own storage tests (pkg/tests/test_storage.py).

The device kernels behind pixels_to_blocks / blocks_to_image / decode are
checked in test_gpu_storage.py.
"""

import os
import struct

import numpy as np
import pytest

import cases
import oracle
from conftest import GOLDEN
from paper_0910_4711_b200 import Codebook, EncodedStream, FormatError, UsageError
from paper_0910_4711_b200 import storage


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLDEN, "storage.npz"))


# ---------------------------------------------------------------------------
# oracle pinning
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("i", range(len(cases.image_cases())))
def test_oracle_blocks_match_reference(gold, i):
    px, b = cases.image_cases()[i]
    got = oracle.pixels_to_blocks(px, b)
    assert got.dtype == np.float64
    assert got.tobytes() == gold[f"img{i}_blocks"].tobytes()


@pytest.mark.parametrize("i", range(len(cases.image_cases())))
def test_oracle_raster_matches_reference(gold, i):
    px, b = cases.image_cases()[i]
    h, w = px.shape
    vec = gold[f"img{i}_blocks"]
    header = len(b"P5\n%d %d\n255\n" % (w, h))
    ident = oracle.blocks_to_pixels(vec, h, w, b)
    assert ident.tobytes() == gold[f"img{i}_pgm_identity"].tobytes()[header:]
    pert = oracle.blocks_to_pixels(cases.raster_vectors(vec, 100 + i), h, w, b)
    assert pert.tobytes() == gold[f"img{i}_pgm"].tobytes()[header:]


@pytest.mark.parametrize("i", range(len(cases.decode_cases())))
def test_oracle_decode_matches_reference(gold, i):
    c = cases.decode_cases()[i]
    assert oracle.decode(c["idx"], c["cb"]).tobytes() == gold[f"dec{i}_rows"].tobytes()


@pytest.mark.parametrize("i", range(len(cases.distortion_cases())))
def test_oracle_distortion_matches_reference(gold, i):
    c = cases.distortion_cases()[i]
    assert oracle.reconstruction_distortion(c["a"], c["b"], c["metric"]) == float(gold[f"dist{i}_total"])


# ---------------------------------------------------------------------------
# VQCB / VQEN: byte images equal the reference's files
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("i", range(len(cases.decode_cases())))
def test_codebook_and_stream_bytes_match_reference(gold, i, tmp_path):
    c = cases.decode_cases()[i]
    cb = Codebook(c["cb"])
    for metric in ("squared_euclidean", "euclidean"):
        want = gold[f"dec{i}_vqcb_{metric}"].tobytes()
        assert storage.codebook_bytes(cb, metric) == want
        path = tmp_path / f"cb_{metric}.vqcb"
        storage.save_codebook(cb, metric, path)
        assert path.read_bytes() == want
        back, m = storage.load_codebook(path)
        assert m == metric and back.codevectors.tobytes() == cb.codevectors.tobytes()
    stream = EncodedStream(cb.size, cb.k, c["idx"])
    want = gold[f"dec{i}_vqen"].tobytes()
    path = tmp_path / "s.vqen"
    storage.save_encoded(stream, path)
    assert path.read_bytes() == want
    back = storage.load_encoded(path)
    assert (back.codebook_size, back.dimension) == (cb.size, cb.k)
    assert back.indices.dtype == np.uint32 and back.indices.tobytes() == stream.indices.tobytes()


def test_codebook_roundtrip_keeps_signed_zero_and_subnormals(tmp_path):
    rows = np.random.default_rng(127).normal(size=(16, 5))
    rows[0, 0] = -0.0
    rows[1, 1] = 5e-324
    path = tmp_path / "cb.vqcb"
    storage.save_codebook(Codebook(rows), "euclidean", path)
    loaded, metric = storage.load_codebook(path)
    assert metric == "euclidean" and loaded.codevectors.tobytes() == rows.tobytes()


def test_codebook_format_errors(tmp_path):
    path = tmp_path / "bad.vqcb"
    path.write_bytes(b"XXXX" + b"\x00" * 32)
    with pytest.raises(FormatError, match="magic"):
        storage.load_codebook(path)
    path.write_bytes(b"VQ")
    with pytest.raises(FormatError, match="truncated header"):
        storage.load_codebook(path)
    path.write_bytes(storage.CODEBOOK_MAGIC + struct.pack("<III", 99, 1, 1) + b"\x00" * 9)
    with pytest.raises(FormatError, match="version"):
        storage.load_codebook(path)
    path.write_bytes(storage.CODEBOOK_MAGIC + struct.pack("<III", 1, 0, 1) + b"\x00")
    with pytest.raises(FormatError, match="invalid codebook shape"):
        storage.load_codebook(path)
    path.write_bytes(storage.CODEBOOK_MAGIC + struct.pack("<III", 1, 1, 1) + struct.pack("<d", 1.0) + b"\x07")
    with pytest.raises(FormatError, match="metric tag"):
        storage.load_codebook(path)
    path.write_bytes(storage.CODEBOOK_MAGIC + struct.pack("<III", 1, 1, 1) + struct.pack("<d", np.inf) + b"\x00")
    with pytest.raises(FormatError, match="non-finite"):
        storage.load_codebook(path)
    blob = storage.codebook_bytes(Codebook(np.ones((4, 3))), "squared_euclidean")
    path.write_bytes(blob[: 16 + 3 * 3 * 8] + blob[-1:])
    with pytest.raises(FormatError, match="size mismatch"):
        storage.load_codebook(path)
    with pytest.raises(UsageError):
        storage.save_codebook(Codebook([(1.0,)]), "manhattan", tmp_path / "x.vqcb")


def test_encoded_format_errors(tmp_path):
    path = tmp_path / "bad.vqen"
    path.write_bytes(b"NOPE" + b"\x00" * 24)
    with pytest.raises(FormatError, match="magic"):
        storage.load_encoded(path)
    storage.save_encoded(EncodedStream(8, 2, [1, 2, 3]), path)
    path.write_bytes(path.read_bytes()[:-2])
    with pytest.raises(FormatError, match="size mismatch"):
        storage.load_encoded(path)
    header = storage.ENCODED_MAGIC + struct.pack("<IIIQ", 1, 4, 2, 2)
    path.write_bytes(header + struct.pack("<II", 1, 9))
    with pytest.raises(FormatError, match="index 9"):
        storage.load_encoded(path)
    path.write_bytes(storage.ENCODED_MAGIC + struct.pack("<IIIQ", 1, 0, 2, 0))
    with pytest.raises(FormatError):
        storage.load_encoded(path)  # EncodedStream's UsageError re-raised as FormatError
    storage.save_encoded(EncodedStream(8, 2, np.empty(0, dtype=np.uint32)), path)
    assert len(storage.load_encoded(path)) == 0


# ---------------------------------------------------------------------------
# PGM + grid
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("i", range(len(cases.image_cases())))
def test_pgm_bytes_match_reference(gold, i):
    px, _ = cases.image_cases()[i]
    data = storage.pgm_bytes(px)
    assert data == gold[f"img{i}_pgmbytes"].tobytes()
    assert np.array_equal(storage.parse_pgm(data), px)


def test_pgm_header_rules():
    assert storage.parse_pgm(b"P5\n# a comment\n3 2\n# another\n255\n" + bytes(6)).shape == (2, 3)
    with pytest.raises(FormatError, match="P5"):
        storage.parse_pgm(b"P2\n2 2\n255\n0 0 0 0")
    with pytest.raises(FormatError, match="maxval"):
        storage.parse_pgm(b"P5\n2 2\n65535\n" + bytes(8))
    with pytest.raises(FormatError, match="truncated"):
        storage.parse_pgm(b"P5\n4 4\n255\n" + bytes(10))
    with pytest.raises(FormatError, match="trailing"):
        storage.parse_pgm(b"P5\n2 2\n255\n" + bytes(5))
    with pytest.raises(FormatError, match="not an integer"):
        storage.parse_pgm(b"P5\nx 2\n255\n")
    with pytest.raises(FormatError, match="positive"):
        storage.parse_pgm(b"P5\n0 2\n255\n")
    with pytest.raises(FormatError, match="truncated PGM header"):
        storage.parse_pgm(b"P5\n2")
    with pytest.raises(UsageError):
        storage.pgm_bytes(np.zeros(4, dtype=np.uint8))


def test_block_grid_geometry(gold):
    for i, (px, b) in enumerate(cases.image_cases()):
        g = storage.BlockGrid(width=px.shape[1], height=px.shape[0], block=b)
        assert [g.width, g.height, g.block, g.count, g.k] == gold[f"img{i}_grid"].tolist()
    with pytest.raises(UsageError):
        storage.BlockGrid(width=0, height=1, block=1)
    with pytest.raises(UsageError):
        storage.BlockGrid(width=1, height=1, block=0)
