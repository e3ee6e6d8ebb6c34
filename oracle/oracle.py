"""CPU oracle for the LBG hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker (and the CPU baseline arm of bench.py).
The product package ``paper_0910_4711_b200`` never imports it; only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may.

It restates the reference's LBG design loop and entry points
(arxiv/paper_0910_4711, ``pkg/src/vqkit``) over the C restatement of the
numba kernels in ``vq_oracle.c``:

* :func:`lbg_train`           <- ``core.lbg_train``          (core.py:366-430)
* :func:`parallel_lbg_train`  <- ``parallel.parallel_lbg_train`` (parallel.py:256-329)
* :func:`assign_cells`        <- ``core.assign_cells``       (core.py:292-316)
* :func:`encode`              <- ``codec.encode``            (codec.py:62-93)
* :func:`update_codebook`     <- ``core.update_codebook``    (core.py:319-339)
* :func:`split_rows`          <- ``core._split_rows``        (core.py:277-281)
* :func:`convergence_check`   <- ``core.convergence_check``  (core.py:342-356)
* :func:`partition_training`  <- ``parallel.partition_training`` (parallel.py:93-107)

Pinning: ``tests/test_oracle.py`` checks every function here against the
reference's own known-answer tests (pkg/tests/conftest.py, test_core.py,
test_parallel.py, test_codec.py) and against golden vectors produced by
running the reference itself (``tests/golden/make_golden.py``).

Plain data in, plain data out: float64 row-major arrays, int64 cells.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libvqoracle.so")

SQUARED_EUCLIDEAN = 0
EUCLIDEAN = 1
_METRICS = {"squared_euclidean": SQUARED_EUCLIDEAN, "euclidean": EUCLIDEAN}

_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(
                f"oracle library missing: {_LIB_PATH} (run `make -C oracle` or "
                "__graft_entry__.build())"
            )
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        I = ctypes.c_int
        lib.vqo_assign_range.argtypes = [P, I64, P, I64, I64, I64, I, P, P]
        lib.vqo_assign_range_f32.argtypes = [P, I64, P, I64, I64, I64, I, P, P]
        lib.vqo_update_rows.argtypes = [P, I64, I64, P, P, I64, I64, I64, P, P]
        lib.vqo_pair_distance.argtypes = [P, P, I64, I]
        lib.vqo_pair_distance.restype = ctypes.c_double
        lib.vqo_column_sums.argtypes = [P, I64, I64, P]
        lib.vqo_sum_inorder.argtypes = [P, I64]
        lib.vqo_sum_inorder.restype = ctypes.c_double
        lib.vqo_assign_parallel.argtypes = [P, P, I64, I64, P, I64, I, I, P, P]
        lib.vqo_update_parallel.argtypes = [P, I64, I64, P, P, I64, I, P, P]
        lib.vqo_max_threads.restype = ctypes.c_int
        lib.vqo_gmm_rows.argtypes = [P, P, P, I64, I64, I64, I64, ctypes.c_uint64, P]
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def metric_code(metric) -> int:
    if isinstance(metric, int):
        return metric
    return _METRICS[metric]


def max_threads() -> int:
    return int(_load().vqo_max_threads())


# ---------------------------------------------------------------------------
# kernel restatements (_kernels.py)
# ---------------------------------------------------------------------------

def assign_range(vectors, codebook, start, stop, metric, out_cells, out_dists):
    """_kernels.assign_range (_kernels.py:18-36)."""
    v = _f64(vectors)
    cb = _f64(codebook)
    _load().vqo_assign_range(_p(v), v.shape[1], _p(cb), cb.shape[0], start, stop,
                             metric_code(metric), _p(out_cells), _p(out_dists))


def update_rows(vectors, cells, old_codebook, worker, stride, out_codebook, out_counts):
    """_kernels.update_rows (_kernels.py:39-66)."""
    v = _f64(vectors)
    c = np.ascontiguousarray(cells, dtype=np.int64)
    cb = _f64(old_codebook)
    _load().vqo_update_rows(_p(v), v.shape[0], v.shape[1], _p(c), _p(cb), cb.shape[0],
                            worker, stride, _p(out_codebook), _p(out_counts))


def pair_distance(a, b, metric) -> float:
    """_kernels.pair_distance (_kernels.py:69-78)."""
    va, vb = _f64(a), _f64(b)
    return float(_load().vqo_pair_distance(_p(va), _p(vb), va.shape[0], metric_code(metric)))


def column_sums(vectors) -> np.ndarray:
    """_kernels.column_sums (_kernels.py:81-89)."""
    v = _f64(vectors)
    out = np.empty(v.shape[1], dtype=np.float64)
    _load().vqo_column_sums(_p(v), v.shape[0], v.shape[1], _p(out))
    return out


def sum_inorder(values) -> float:
    """_kernels.sum_inorder (_kernels.py:92-98)."""
    v = _f64(values)
    return float(_load().vqo_sum_inorder(_p(v), v.shape[0]))


# ---------------------------------------------------------------------------
# engine restatements (core.py / parallel.py / codec.py)
# ---------------------------------------------------------------------------

def partition_training(m: int, workers: int) -> list[tuple[int, int]]:
    """parallel.partition_training (parallel.py:93-107)."""
    base, extra = divmod(m, workers)
    ranges, cursor = [], 0
    for rho in range(workers):
        size = base + (1 if rho < extra else 0)
        ranges.append((cursor, cursor + size))
        cursor += size
    return ranges


def split_rows(rows: np.ndarray, delta: float) -> np.ndarray:
    """core._split_rows (core.py:277-281): row i -> 2i (+delta), 2i+1 (-delta)."""
    out = np.empty((rows.shape[0] * 2, rows.shape[1]), dtype=np.float64)
    out[0::2] = rows + delta
    out[1::2] = rows - delta
    return out


def convergence_check(td_prev: float, td_cur: float, epsilon: float) -> bool:
    """core.convergence_check (core.py:342-356), minus the error raising."""
    if math.isinf(td_prev):
        return False
    if td_prev == 0.0:
        return True
    return (td_prev - td_cur) / td_prev <= epsilon


def assign_all(vectors, codebook, metric=SQUARED_EUCLIDEAN, workers: int = 1,
               vectors32=None):
    """Allocation over all rows -> (cells int64[m], dists f64[m]).  With
    workers > 1 it is the OpenMP master/slave phase (parallel.py:135-141)."""
    cb = _f64(codebook)
    if vectors32 is not None:
        v32 = np.ascontiguousarray(vectors32, dtype=np.float32)
        m, dim = v32.shape
        v = None
    else:
        v = _f64(vectors)
        v32 = None
        m, dim = v.shape
    cells = np.empty(m, dtype=np.int64)
    dists = np.empty(m, dtype=np.float64)
    if m == 0:
        return cells, dists
    _load().vqo_assign_parallel(
        _p(v) if v is not None else None, _p(v32) if v32 is not None else None,
        m, dim, _p(cb), cb.shape[0], metric_code(metric), max(1, int(workers)),
        _p(cells), _p(dists))
    return cells, dists


def update_all(vectors, cells, codebook, workers: int = 1):
    """Updation over all codevectors -> (new_rows, counts).  workers > 1 is
    the round-robin phase (parallel.py:144-154)."""
    v = _f64(vectors)
    cb = _f64(codebook)
    c = np.ascontiguousarray(cells, dtype=np.int64)
    new_rows = np.empty_like(cb)
    counts = np.zeros(cb.shape[0], dtype=np.int64)
    _load().vqo_update_parallel(_p(v), v.shape[0], v.shape[1], _p(c), _p(cb), cb.shape[0],
                                max(1, int(workers)), _p(new_rows), _p(counts))
    return new_rows, counts


def assign_cells(chunk, codebook, metric=SQUARED_EUCLIDEAN):
    """core.assign_cells (core.py:292-316) -> (cells int64, in-order total)."""
    cells, dists = assign_all(chunk, codebook, metric)
    return cells, sum_inorder(dists)


def encode(data, codebook, workers: int = 1) -> np.ndarray:
    """codec.encode (codec.py:62-93) -> uint32 indices (metric forced squared)."""
    cells, _ = assign_all(data, codebook, SQUARED_EUCLIDEAN, workers)
    return cells.astype(np.uint32)


def update_codebook(vectors, cells, codebook):
    """core.update_codebook (core.py:319-339) -> (new rows, empty count)."""
    new_rows, counts = update_all(vectors, cells, codebook)
    return new_rows, int(np.count_nonzero(counts == 0))


@dataclass
class Pass:
    """One allocation pass as seen by the oracle (for teacher forcing)."""

    size: int
    iteration: int
    codebook: np.ndarray      # codebook fed to the allocation
    td: float
    counts: np.ndarray        # bincount of the cells (minlength=size)
    updated: np.ndarray | None  # codebook after the update (None on convergence)
    empty_cells: int


@dataclass
class Result:
    codebook: np.ndarray
    total: float
    history: list[tuple[int, int, float, int]] = field(default_factory=list)
    warnings: list[str] = field(default_factory=list)
    per_worker: list[float] = field(default_factory=list)
    passes: list[Pass] = field(default_factory=list)
    final_cells: np.ndarray | None = None
    final_dists: np.ndarray | None = None


def _max_iter_warning(level_size: int, limit: int) -> str:
    # core.py:359-363
    return (
        f"codebook level {level_size} stopped after {limit} iterations "
        f"without meeting the distortion threshold"
    )


def lbg_train(vectors, target_size: int, epsilon: float = 1e-3, delta: float = 0.01,
              workers: int = 1, max_iterations_per_level: int = 100,
              metric=SQUARED_EUCLIDEAN, record: bool = False, vectors32=None,
              progress=None) -> Result:
    """core.lbg_train (core.py:366-430) / parallel.parallel_lbg_train
    (parallel.py:256-329).  ``workers`` only changes the thread count and the
    per_worker chunks; the result is bit-identical for every value, as in
    the reference.  ``record`` keeps every pass for teacher forcing."""
    v = _f64(vectors) if vectors32 is None else np.asarray(vectors32, np.float32).astype(np.float64)
    code = metric_code(metric)
    m = v.shape[0]
    rows = (column_sums(v) / m).reshape(1, -1)
    history, warnings, passes = [], [], []
    cells = dists = None
    size = 1
    started = time.perf_counter()
    while size < target_size:
        rows = split_rows(rows, delta)
        size *= 2
        td_prev = math.inf
        converged = False
        for iteration in range(1, max_iterations_per_level + 1):
            cells, dists = assign_all(v, rows, code, workers, vectors32=vectors32)
            td = sum_inorder(dists)
            if convergence_check(td_prev, td, epsilon):
                history.append((size, iteration, td, 0))
                if record:
                    passes.append(Pass(size, iteration, rows.copy(), td,
                                       np.bincount(cells, minlength=size), None, 0))
                converged = True
                break
            new_rows, counts = update_all(v, cells, rows, workers)
            empty = int(np.count_nonzero(counts == 0))
            history.append((size, iteration, td, empty))
            if record:
                passes.append(Pass(size, iteration, rows.copy(), td, counts.copy(),
                                   new_rows.copy(), empty))
            rows = new_rows
            td_prev = td
            if progress is not None:
                progress(size, iteration, td, time.perf_counter() - started)
        if not converged:
            warnings.append(_max_iter_warning(size, max_iterations_per_level))
    if history:
        total = history[-1][2]
    else:
        cells, dists = assign_all(v, rows, code, workers, vectors32=vectors32)
        total = sum_inorder(dists)
    per_worker = [sum_inorder(dists[lo:hi]) for lo, hi in partition_training(m, max(1, workers))]
    return Result(rows, total, history, warnings, per_worker, passes, cells, dists)


def top2_gaps(vectors, codebook) -> np.ndarray:
    """Relative FP64 gap (d2 - d1) / d2 between the nearest and second-nearest
    codevector in the reference's arithmetic (near-tie audit, BASELINE
    north_star: ties are rows with relative gap < 1e-6).  numpy restatement
    of _kernels.py:25-29 with the same per-op rounding (no FMA in numpy)."""
    v = _f64(vectors)
    cb = _f64(codebook)
    m = v.shape[0]
    out = np.empty(m, dtype=np.float64)
    step = max(1, (1 << 22) // max(1, cb.shape[0] * v.shape[1]))
    for lo in range(0, m, step):
        x = v[lo:lo + step]
        d = np.zeros((x.shape[0], cb.shape[0]), dtype=np.float64)
        for l in range(v.shape[1]):
            diff = x[:, l:l + 1] - cb[None, :, l]
            d = d + diff * diff
        if cb.shape[0] < 2:
            out[lo:lo + step] = np.inf
            continue
        part = np.partition(d, 1, axis=1)
        d1, d2 = part[:, 0], part[:, 1]
        with np.errstate(divide="ignore", invalid="ignore"):
            out[lo:lo + step] = np.where(d2 > 0, (d2 - d1) / d2, 0.0)
    return out


# ---------------------------------------------------------------------------
# data formats either side of the path
# ---------------------------------------------------------------------------
# * pixels_to_blocks          <- storage.pixels_to_blocks (storage.py:281-293)
# * blocks_to_pixels          <- storage.blocks_to_image raster (storage.py:296-311)
# * decode                    <- codec.decode (codec.py:96-114)
# * reconstruction_distortion <- codec.reconstruction_distortion (codec.py:135-156)
# Restated with explicit index maps (block v = (by, bx), element q = (r, c)),
# not the reference's reshape/swapaxes chain.

def gmm_rows(means, sigmas, cum_weights, rows: int, seed: int, row_offset: int = 0) -> np.ndarray:
    """Host restatement of the device Gaussian-mixture generator
    (csrc/gmm.cu gmm_rows_kernel; vq_oracle.c vqo_gmm_rows): float32 rows
    [row_offset, row_offset + rows) of the set drawn with ``seed``."""
    m = np.ascontiguousarray(means, dtype=np.float32)
    sg = np.ascontiguousarray(sigmas, dtype=np.float32)
    cw = None if cum_weights is None else np.ascontiguousarray(cum_weights, dtype=np.float64)
    out = np.empty((rows, m.shape[1]), dtype=np.float32)
    _load().vqo_gmm_rows(_p(m), _p(sg), None if cw is None else _p(cw), m.shape[0], rows, m.shape[1],
                         row_offset, seed, _p(out))
    return out


def pixels_to_blocks(pixels, block: int) -> np.ndarray:
    """float64 [ceil(h/b) * ceil(w/b)][b*b]; out-of-image samples take the
    nearest edge pixel (np.pad mode "edge" == clamping the coordinates)."""
    px = np.asarray(pixels, dtype=np.uint8)
    h, w = px.shape
    bc, br = -(-w // block), -(-h // block)
    by, bx, r, c = np.meshgrid(np.arange(br), np.arange(bc), np.arange(block), np.arange(block),
                               indexing="ij")
    y = np.minimum(by * block + r, h - 1)
    x = np.minimum(bx * block + c, w - 1)
    return px[y, x].reshape(br * bc, block * block).astype(np.float64)


def blocks_to_pixels(vectors, height: int, width: int, block: int) -> np.ndarray:
    """uint8 [h][w]: pixel (y, x) is element (y % b, x % b) of block
    (y // b, x // b), clamped to [0, 255] and rounded half up."""
    v = np.asarray(vectors, dtype=np.float64)
    bc = -(-width // block)
    y, x = np.meshgrid(np.arange(height), np.arange(width), indexing="ij")
    vals = v[(y // block) * bc + x // block, (y % block) * block + x % block]
    return np.floor(np.clip(vals, 0.0, 255.0) + 0.5).astype(np.uint8)


def decode(indices, codebook) -> np.ndarray:
    cb = _f64(codebook)
    idx = np.asarray(indices, dtype=np.int64)
    if idx.size and (idx.max() >= cb.shape[0] or idx.min() < 0):
        raise ValueError("corrupt stream")
    return cb[idx]


def reconstruction_distortion(a, b, metric=SQUARED_EUCLIDEAN) -> float:
    """Per-row pair_distance (vq_oracle.c, _kernels.py:69-78) summed in input
    order (sum_inorder, _kernels.py:92-98)."""
    a, b = _f64(a), _f64(b)
    # column by column over all rows: per row the same ascending-c sequence of
    # separately rounded ops as the scalar kernel (numpy never contracts to FMA)
    d = np.zeros(a.shape[0], dtype=np.float64)
    for c in range(a.shape[1]):
        diff = a[:, c] - b[:, c]
        d = d + diff * diff
    if metric_code(metric) == 1:
        d = np.sqrt(d)
    return sum_inorder(d) if d.size else 0.0
