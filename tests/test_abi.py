"""The drop-in boundary on a CPU box: libvqb200.so (built for sm_100a) loads,
exports every entry point include/vqb200.h declares, and the product package
fails loudly -- never silently on the CPU -- when no device or no library is
there.  No compute call is made without a GPU."""

import ast
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vqb200.h")
PKG = os.path.join(ROOT, "paper_0910_4711_b200")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vqb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("vqb_assign_range", "vqb_update_rows", "vqb_column_sums", "vqb_sum_inorder",
                 "vqb_pair_distance", "vqb_open", "vqb_train", "vqb_assign", "vqb_update",
                 "vqb_close", "vqb_encode_f32", "vqb_last_error"):
        assert must in names


def test_library_loads_and_exports_every_declared_symbol():
    from paper_0910_4711_b200 import _lib

    lib = _lib.lib()
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(raw, name), f"{name} declared in include/vqb200.h but not exported"
    # every symbol the ctypes binding types is declared in the header too
    assert lib.vqb_version() >= 1


def test_library_is_sm100a_code():
    from paper_0910_4711_b200 import _lib
    import shutil
    import subprocess

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_is_an_error_not_a_fallback():
    from paper_0910_4711_b200 import _lib
    import paper_0910_4711_b200 as vq

    if _lib.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(vq.InternalError):
        _lib.require_device()
    with pytest.raises(vq.InternalError):
        vq.encode(np.zeros((4, 2), np.float32), vq.Codebook(np.zeros((2, 2))))
    with pytest.raises(vq.InternalError):
        vq.lbg_train(vq.TrainingSet(np.zeros((8, 2))), vq.LbgConfig(target_size=2))


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_0910_4711_b200 import _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "libvqb200.so"))
    with pytest.raises(ImportError, match="no CPU fallback"):
        _lib.lib()


def test_validation_errors_before_any_device_call():
    import paper_0910_4711_b200 as vq

    with pytest.raises(vq.ConfigError):
        vq.LbgConfig(target_size=3)
    with pytest.raises(vq.ConfigError):
        vq.LbgConfig(target_size=4, epsilon=-1)
    with pytest.raises(vq.UsageError):
        vq.TrainingSet(np.array([[1.0, np.nan]]))
    with pytest.raises(vq.UsageError, match="dimension"):
        vq.encode(np.zeros((4, 2)), vq.Codebook(np.zeros((2, 3))))
    with pytest.raises(vq.UsageError):
        vq.assign_cells(np.empty((0, 3)), vq.Codebook(np.zeros((2, 3))))
    assert len(vq.encode(np.empty((0, 3)), vq.Codebook(np.zeros((2, 3))))) == 0
    assert vq.convergence_check(100.0, 99.99, 1e-3) is True
    with pytest.raises(vq.DomainError):
        vq.convergence_check(-1.0, 1.0, 1e-3)


def test_product_never_imports_the_oracle():
    """Only tests/, __graft_entry__.smoke() and bench.py may use oracle/."""
    for fn in os.listdir(PKG):
        if not fn.endswith(".py"):
            continue
        tree = ast.parse(open(os.path.join(PKG, fn)).read())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                mods = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                mods = [node.module or ""]
            else:
                continue
            assert not any(m.split(".")[0] in ("oracle", "vqkit") for m in mods), (fn, mods)
    for fn in os.listdir(os.path.join(PKG, "csrc")):
        src = open(os.path.join(PKG, "csrc", fn)).read()
        assert "vq_oracle" not in src and "vqo_" not in src, fn


def test_every_reference_export_exists():
    """Every name of vqkit.__all__ (pkg/src/vqkit/__init__.py:79-135) is
    importable from the package (the GPU sweep harness stands in for the
    thread sweep of bench.py)."""
    import paper_0910_4711_b200 as vq

    for name in ("AmdahlParams", "BenchRecord", "amdahl_speedup", "run_sweep", "speedup_report",
                 "synthetic_training_set", "write_bench_csv", "load_training_csv", "save_vectors_csv",
                 "BlockGrid", "blocks_to_image", "image_to_blocks", "load_codebook", "load_encoded",
                 "parse_pgm", "pgm_bytes", "pixels_to_blocks", "read_pgm", "save_codebook",
                 "save_encoded", "RateReport", "rate", "decode", "reconstruction_distortion"):
        assert hasattr(vq, name) and name in vq.__all__, name


def test_public_names_match_the_reference_surface():
    """The hot-path names of vqkit.__all__ (pkg/src/vqkit/__init__.py:79-135)."""
    import paper_0910_4711_b200 as vq

    for name in ("TrainingSet", "Codebook", "CellTable", "LevelIteration", "DistortionStats",
                 "LbgConfig", "lbg_train", "parallel_lbg_train", "encode", "assign_cells",
                 "update_codebook", "split_codebook", "convergence_check", "nearest_codevector",
                 "centroid", "distance", "partition_training", "parallel_assign", "integrate",
                 "parallel_update", "ChunkPlan", "UpdateAssignment", "EncodedStream",
                 "VqError", "UsageError", "ConfigError", "DomainError", "FormatError",
                 "InternalError", "SQUARED_EUCLIDEAN", "EUCLIDEAN", "decode",
                 "reconstruction_distortion", "BlockGrid", "pixels_to_blocks", "blocks_to_image",
                 "image_to_blocks", "parse_pgm", "pgm_bytes", "read_pgm", "save_codebook",
                 "load_codebook", "save_encoded", "load_encoded"):
        assert hasattr(vq, name), name
        assert name in vq.__all__, name
