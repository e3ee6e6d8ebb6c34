"""The ``vq`` command line (paper_0910_4711_b200/cli.py), modelled on the
reference's pkg/tests/test_cli.py: exit-code contract (0 ok, 1 usage, 2 data),
output lines and files.  Paths that reach the device are marked gpu; the
argument / file-format error paths run on CPU."""

import numpy as np
import pytest

from paper_0910_4711_b200 import Codebook, load_codebook, load_encoded, parse_pgm, pgm_bytes
from paper_0910_4711_b200 import storage
from paper_0910_4711_b200.cli import main

TRACE_CSV = "0,0\n0,1\n4,0\n4,1\n"  # the reference's trace (conftest.py:7-26)


@pytest.fixture
def trace_csv(tmp_path):
    path = tmp_path / "trace.csv"
    path.write_text(TRACE_CSV)
    return path


def run(*argv):
    return main([str(a) for a in argv])


def _gradient_pgm(path, width=32, height=32):
    x = np.arange(width, dtype=np.float64)
    y = np.arange(height, dtype=np.float64)[:, None]
    img = np.floor((x + y) * 255.0 / (width + height - 2) + 0.5).astype(np.uint8)
    path.write_bytes(pgm_bytes(img))
    return img


# ---------------------------------------------------------------------------
# CPU: argument and format errors never reach the device
# ---------------------------------------------------------------------------

def test_unknown_flag_and_no_command(capsys):
    assert run("train", "--frobnicate") == 1
    assert run() == 1
    assert "usage" in capsys.readouterr().out.lower()


def test_train_rejects_non_power_of_two(tmp_path, trace_csv, capsys):
    assert run("train", "--input", trace_csv, "--codebook-size", 3, "--out", tmp_path / "x") == 1
    assert "power of two" in capsys.readouterr().err


def test_missing_input_is_data_error(tmp_path):
    assert run("train", "--input", tmp_path / "nope.csv", "--codebook-size", 2,
               "--out", tmp_path / "x.vqcb") == 2


def test_rate_and_corrupt_codebook(tmp_path, capsys):
    cb = tmp_path / "cb.vqcb"
    storage.save_codebook(Codebook(np.random.default_rng(1).random((128, 10))), "euclidean", cb)
    assert run("rate", "--codebook", cb) == 0
    out = capsys.readouterr().out
    assert "0.7 bits/sample" in out and "7 bits/vector" in out and "metric euclidean" in out
    bad = tmp_path / "bad.vqcb"
    bad.write_bytes(b"GARBAGE!" * 4)
    assert run("rate", "--codebook", bad) == 2
    assert "magic" in capsys.readouterr().err


def test_bench_bad_sweep_list_is_usage_error(tmp_path):
    assert run("bench", "--sizes", "8,x", "--gpus", "1", "--out", tmp_path / "b.csv") == 1
    assert run("bench", "--synthetic", "1,2", "--out", tmp_path / "b.csv") == 1


def test_vq_threads_env_validation(tmp_path, trace_csv, monkeypatch):
    monkeypatch.setenv("VQ_THREADS", "zero")
    assert run("train", "--input", trace_csv, "--codebook-size", 2, "--out", tmp_path / "c") == 1
    monkeypatch.setenv("VQ_THREADS", "0")
    assert run("train", "--input", trace_csv, "--codebook-size", 2, "--out", tmp_path / "c") == 1


def test_csv_loader_messages(tmp_path):
    p = tmp_path / "r.csv"
    p.write_text("1,2\n1,2,3\n")
    with pytest.raises(storage.FormatError, match="row 2"):
        storage.load_training_csv(p)
    p.write_text("1,2\n3,oops\n")
    with pytest.raises(storage.FormatError, match="row 2, column 2"):
        storage.load_training_csv(p)
    p.write_text("1,nan\n")
    with pytest.raises(storage.FormatError, match="non-finite"):
        storage.load_training_csv(p)
    p.write_text("")
    with pytest.raises(storage.FormatError, match="no data"):
        storage.load_training_csv(p)
    rows = np.random.default_rng(113).normal(size=(7, 3))
    storage.save_vectors_csv(rows, p)
    assert storage.load_training_csv(p).vectors.tobytes() == rows.tobytes()


# ---------------------------------------------------------------------------
# GPU: the flows
# ---------------------------------------------------------------------------

@pytest.mark.gpu
def test_train_writes_expected_codebook(tmp_path, trace_csv, capsys):
    out, hist = tmp_path / "cb.vqcb", tmp_path / "hist.csv"
    assert run("train", "--input", trace_csv, "--codebook-size", 2, "--delta", 0.5,
               "--threads", 1, "--out", out, "--history", hist) == 0
    cb, metric = load_codebook(out)
    assert metric == "squared_euclidean"
    assert cb.codevectors.tolist() == [[4.0, 0.5], [0.0, 0.5]]
    lines = hist.read_text().strip().split("\n")
    assert lines[0] == "level_size,iteration,td,empty_cells,seconds"
    assert len(lines) == 4 and lines[1].startswith("2,1,11.0,")
    captured = capsys.readouterr().out
    assert "total 1" in captured and "bits/sample" in captured


@pytest.mark.gpu
def test_train_threads_do_not_change_file_bytes(tmp_path):
    big = tmp_path / "big.csv"
    rows = np.random.default_rng(137).random((300, 5))
    big.write_text("\n".join(",".join(repr(float(v)) for v in r) for r in rows))
    out1, out4 = tmp_path / "p1.vqcb", tmp_path / "p4.vqcb"
    assert run("train", "--input", big, "--codebook-size", 16, "--threads", 1, "--out", out1) == 0
    assert run("train", "--input", big, "--codebook-size", 16, "--threads", 4, "--out", out4) == 0
    assert out1.read_bytes() == out4.read_bytes()


@pytest.mark.gpu
def test_encode_decode_roundtrip_and_mismatch(tmp_path, trace_csv, capsys):
    cb2, cb4 = tmp_path / "cb2.vqcb", tmp_path / "cb4.vqcb"
    assert run("train", "--input", trace_csv, "--codebook-size", 2, "--delta", 0.5, "--out", cb2) == 0
    assert run("train", "--input", trace_csv, "--codebook-size", 4, "--out", cb4) == 0
    enc = tmp_path / "t.vqen"
    assert run("encode", "--input", trace_csv, "--codebook", cb2, "--threads", 2, "--out", enc) == 0
    assert load_encoded(enc).indices.tolist() == [1, 1, 0, 0]
    dec = tmp_path / "recon.csv"
    assert run("decode", "--input", enc, "--codebook", cb2, "--out", dec) == 0
    assert storage.load_training_csv(dec).vectors.tolist() == [[0.0, 0.5], [0.0, 0.5], [4.0, 0.5], [4.0, 0.5]]
    capsys.readouterr()
    assert run("decode", "--input", enc, "--codebook", cb4, "--out", tmp_path / "y.csv") == 1
    assert "codevectors" in capsys.readouterr().err


@pytest.mark.gpu
def test_image_pipeline(tmp_path, capsys):
    img = tmp_path / "in.pgm"
    original = _gradient_pgm(img)
    cb = tmp_path / "img.vqcb"
    assert run("image-train", "--image", img, "--block", 4, "--codebook-size", 16, "--out", cb) == 0
    enc = tmp_path / "img.vqen"
    assert run("image-encode", "--image", img, "--codebook", cb, "--out", enc, "--report") == 0
    out = capsys.readouterr().out
    assert "reconstruction distortion" in out and "--width 32 --height 32" in out
    dec = tmp_path / "out.pgm"
    assert run("image-decode", "--input", enc, "--codebook", cb, "--width", 32, "--height", 32,
               "--out", dec) == 0
    decoded = parse_pgm(dec.read_bytes())
    assert decoded.shape == original.shape
    # the fused device decode equals the reference's two-step raster of decode
    stream, (codebook, _) = load_encoded(enc), load_codebook(cb)
    rows = codebook.codevectors[stream.indices.astype(np.int64)]
    want = np.floor(np.clip(rows, 0, 255) + 0.5).astype(np.uint8).reshape(8, 8, 4, 4)
    assert np.array_equal(decoded, want.swapaxes(1, 2).reshape(32, 32))
    assert run("image-decode", "--input", enc, "--codebook", cb, "--width", 100, "--height", 100,
               "--out", tmp_path / "o.pgm") == 1


@pytest.mark.gpu
def test_image_encode_non_square_codebook(tmp_path, trace_csv, capsys):
    img = tmp_path / "in.pgm"
    _gradient_pgm(img)
    flat = tmp_path / "flat.vqcb"
    run("train", "--input", trace_csv, "--codebook-size", 2, "--out", flat)
    assert run("image-encode", "--image", img, "--codebook", flat, "--out", tmp_path / "x.vqen") == 1
    assert "square" in capsys.readouterr().err


@pytest.mark.gpu
def test_bench_writes_csv_and_speedups(tmp_path, capsys):
    out = tmp_path / "bench.csv"
    assert run("bench", "--synthetic", "80,3,7", "--sizes", "2,4", "--gpus", "1", "--repeats", 1,
               "--out", out) == 0
    lines = out.read_text().strip().split("\n")
    assert lines[0].startswith("# synthetic m=80 k=3 seed=7")
    assert lines[1] == "n,p,m,k,seconds,td,iterations" and len(lines) == 4
    stdout = capsys.readouterr().out
    assert "Amdahl prediction" in stdout and "speedup 1.00x" in stdout


@pytest.mark.gpu
def test_vq_threads_env_override(tmp_path, trace_csv, monkeypatch, capsys):
    monkeypatch.setenv("VQ_THREADS", "2")
    assert run("train", "--input", trace_csv, "--codebook-size", 2, "--out", tmp_path / "cb") == 0
    assert "2 worker(s)" in capsys.readouterr().out
