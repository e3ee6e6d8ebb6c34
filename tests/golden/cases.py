"""Seeded input cases shared by the golden generator (run against the
reference) and the parity tests (run against the oracle and the GPU path).

Only inputs live here; reference outputs are in tests/golden/small.npz.
The shapes follow the reference's own tests (pkg/tests/test_core.py,
test_parallel.py, test_codec.py) plus the BASELINE dimensions (L=16, 64).
"""

from __future__ import annotations

import numpy as np


def _f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def assign_cases():
    out = []
    # 0: the reference's trace (conftest.py:7-26) against its split codebook
    out.append(dict(x=np.array([[0.0, 0.0], [0.0, 1.0], [4.0, 0.0], [4.0, 1.0]]),
                    cb=np.array([[2.5, 1.0], [1.5, 0.0]]), metric=0))
    # 1: tie rule (test_core.py:163-165)
    out.append(dict(x=np.array([[0.0, 0.0]]),
                    cb=np.array([[9.0, 9.0], [1.0, 0.0], [-1.0, 0.0]]), metric=0))
    rng = np.random.default_rng(1001)
    # 2-3: float64 normals (NOT float32-exact), like test_core.py:168-179,247-258
    out.append(dict(x=rng.normal(size=(300, 4)), cb=rng.normal(size=(12, 4)), metric=0))
    out.append(dict(x=rng.normal(size=(257, 7)), cb=rng.normal(size=(33, 7)), metric=1))
    # 4: uniform [0,1) f64 (bench.py:59-62 generator), k=6, S=16
    out.append(dict(x=rng.random((1000, 6)), cb=rng.random((16, 6)), metric=0))
    # 5: L=16 float32 GMM-like rows, K=256
    means = rng.uniform(0, 255, (64, 16))
    lab = rng.integers(0, 64, 4096)
    x = _f32(means[lab] + rng.normal(0, 8, (4096, 16)))
    out.append(dict(x=x, cb=_f32(x[rng.choice(4096, 256, replace=False)] + 0.25), metric=0))
    # 6: L=16 integer pixels with duplicate codevectors (tie-dense), K=64
    x = rng.integers(0, 256, (3000, 16)).astype(np.float64)
    cb = rng.integers(0, 256, (32, 16)).astype(np.float64)
    cb = np.repeat(cb, 2, axis=0)  # every codevector twice -> exact ties, lowest wins
    out.append(dict(x=x, cb=cb, metric=0))
    # 7: L=64 integer pixels, K=512 (cfg3 shape)
    x = rng.integers(0, 256, (2048, 64)).astype(np.float64)
    cb = x[rng.choice(2048, 512, replace=False)] + rng.choice([-0.5, 0.5], (512, 64))
    out.append(dict(x=x, cb=cb, metric=0))
    # 8: L=16, K=4096 (cfg4 shape, codebook larger than one smem tile)
    x = _f32(rng.uniform(0, 255, (2000, 16)))
    cb = _f32(rng.uniform(0, 255, (4096, 16)))
    out.append(dict(x=x, cb=cb, metric=0))
    # 9: K=1 and a single row
    out.append(dict(x=rng.normal(size=(1, 5)), cb=rng.normal(size=(1, 5)), metric=0))
    # 10: L=1, K=2 first-split-like tie-dense case (centroid +- delta)
    x = _f32(rng.uniform(0, 255, (5000, 1)))
    c = x.mean(axis=0, keepdims=True)
    out.append(dict(x=x, cb=np.concatenate([c + 0.01, c - 0.01]), metric=0))
    # 11: L=16 first split of a GMM (K=2, additive delta): the tie-densest point
    means = rng.uniform(0, 255, (128, 16))
    lab = rng.integers(0, 128, 20000)
    x = _f32(means[lab] + rng.normal(0, 10, (20000, 16)))
    c = x.sum(axis=0, keepdims=True) / x.shape[0]
    out.append(dict(x=x, cb=np.concatenate([c + 0.01, c - 0.01]), metric=0))
    # 12: L=64 float32 data, euclidean metric
    x = _f32(rng.uniform(0, 255, (1500, 64)))
    out.append(dict(x=x, cb=_f32(rng.uniform(0, 255, (100, 64))), metric=1))
    # 13: L=32 float32, K=300 (non power of two, generic path)
    x = _f32(rng.normal(50, 20, (2500, 32)))
    out.append(dict(x=x, cb=_f32(rng.normal(50, 20, (300, 32))), metric=0))
    return out


def update_cases():
    out = []
    rng = np.random.default_rng(2002)
    # 0: trace update (test_core.py:265-271)
    out.append(dict(x=np.array([[0.0, 0.0], [0.0, 1.0], [4.0, 0.0], [4.0, 1.0]]),
                    cells=np.array([1, 1, 0, 0], dtype=np.int64),
                    cb=np.array([[2.5, 1.0], [1.5, 0.0]])))
    # 1: empty cell retention (test_core.py:274-279)
    out.append(dict(x=np.array([[0.0, 0.0], [0.0, 1.0], [4.0, 0.0], [4.0, 1.0]]),
                    cells=np.array([0, 0, 0, 0], dtype=np.int64),
                    cb=np.array([[2.5, 1.0], [1.5, 0.0]])))
    # 2: f64 normals (test_core.py:287-298 shape)
    out.append(dict(x=rng.normal(size=(97, 5)), cells=rng.integers(0, 8, 97).astype(np.int64),
                    cb=rng.normal(size=(8, 5))))
    # 3: L=16 float32 data, K=1024 with many empty cells
    x = _f32(rng.uniform(0, 255, (5000, 16)))
    out.append(dict(x=x, cells=rng.integers(0, 700, 5000).astype(np.int64),
                    cb=_f32(rng.uniform(0, 255, (1024, 16)))))
    # 4: L=64 pixels, K=512
    x = rng.integers(0, 256, (4096, 64)).astype(np.float64)
    out.append(dict(x=x, cells=rng.integers(0, 512, 4096).astype(np.int64),
                    cb=rng.uniform(0, 255, (512, 64))))
    # 5: K=2, all rows in two huge cells with tiny and large magnitudes mixed
    x = _f32(np.concatenate([rng.uniform(0, 255, (20000, 16)),
                             rng.uniform(-1e-3, 1e-3, (100, 16))]))
    out.append(dict(x=x, cells=rng.integers(0, 2, x.shape[0]).astype(np.int64),
                    cb=np.zeros((2, 16))))
    return out


def design_cases():
    out = []
    trace = np.array([[0.0, 0.0], [0.0, 1.0], [4.0, 0.0], [4.0, 1.0]])
    # 0: the reference trace (test_core.py:340-347)
    out.append(dict(x=trace, config=dict(target_size=2, epsilon=1e-3, delta=0.5)))
    # 1: euclidean trace (test_core.py:431-437)
    out.append(dict(x=trace, config=dict(target_size=2, delta=0.5,
                                         distortion_metric="euclidean")))
    # 2: target 1 (test_core.py:360-364)
    out.append(dict(x=trace, config=dict(target_size=1)))
    # 3: identical vectors, empty cells (test_core.py:349-357)
    out.append(dict(x=np.tile(np.array([2.5, -1.5]), (5, 1)),
                    config=dict(target_size=2, delta=0.5)))
    rng = np.random.default_rng(3003)
    # 4: iteration guard (test_core.py:367-380)
    out.append(dict(x=rng.random((64, 3)),
                    config=dict(target_size=8, epsilon=0.0, max_iterations_per_level=1)))
    # 5: uniform f64, workers=3 (test_parallel.py:178-192 shape)
    out.append(dict(x=rng.random((200, 6)), config=dict(target_size=16, workers=3)))
    # 6: L=16 float32 GMM, K=64
    means = rng.uniform(0, 255, (48, 16))
    lab = rng.integers(0, 48, 6000)
    x = _f32(means[lab] + rng.normal(0, 6, (6000, 16)))
    out.append(dict(x=x, config=dict(target_size=64, epsilon=1e-4, delta=0.01, workers=4)))
    # 7: L=64 integer pixels, K=32
    x = rng.integers(0, 256, (3000, 64)).astype(np.float64)
    out.append(dict(x=x, config=dict(target_size=32, epsilon=1e-3, delta=0.01)))
    # 8: L=16 pixels, euclidean, K=16
    x = rng.integers(0, 256, (4000, 16)).astype(np.float64)
    out.append(dict(x=x, config=dict(target_size=16, delta=0.01,
                                     distortion_metric="euclidean", workers=2)))
    return out


def encode_cases():
    rng = np.random.default_rng(4004)
    out = []
    cb = rng.normal(size=(13, 4))
    out.append(dict(x=rng.normal(size=(50, 4)), cb=cb, workers=1))
    cb = _f32(rng.uniform(0, 255, (1024, 16)))
    out.append(dict(x=_f32(rng.uniform(0, 255, (20000, 16))), cb=cb, workers=4))
    return out


# ---------------------------------------------------------------------------
# data formats either side of the path (storage.py / codec.py decode)
# ---------------------------------------------------------------------------

def image_cases():
    """(pixels uint8 [h][w], block) -- ragged edges, every block side the band
    kernel specialises (2, 4, 8, 16), sides it does not (1, 3, 5) and a band
    too wide for shared memory (generic path)."""
    rng = np.random.default_rng(5005)
    out = []
    out.append((np.arange(16, dtype=np.uint8).reshape(4, 4), 2))  # test_storage.py:236-241 layout
    out.append((np.array([[1, 2], [3, 4]], dtype=np.uint8), 3))   # edge replication
    out.append((np.array([[7]], dtype=np.uint8), 1))
    grad = ((np.arange(9)[:, None] * 17 + np.arange(17)[None, :] * 5) % 256).astype(np.uint8)
    out.append((grad, 5))
    out.append((rng.integers(0, 256, (7, 13), dtype=np.uint8), 4))
    out.append((rng.integers(0, 256, (48, 64), dtype=np.uint8), 8))
    out.append((rng.integers(0, 256, (37, 70), dtype=np.uint8), 16))
    out.append((rng.integers(0, 256, (65, 33), dtype=np.uint8), 4))
    out.append((rng.integers(0, 256, (11, 10), dtype=np.uint8), 3))
    out.append((rng.integers(0, 256, (5, 3000), dtype=np.uint8), 16))   # band = 48128 B, staged
    out.append((rng.integers(0, 256, (7, 4000), dtype=np.uint8), 16))   # band > 48 KiB: generic
    out.append((rng.integers(0, 256, (31, 29), dtype=np.uint8), 2))
    return out


def raster_vectors(vectors, seed):
    """Block vectors perturbed past both clamps and onto exact .5 ties."""
    rng = np.random.default_rng(seed)
    v = np.asarray(vectors, dtype=np.float64) + rng.normal(0, 40, vectors.shape)
    half = rng.random(vectors.shape) < 0.2
    v[half] = np.floor(v[half]) + 0.5
    return v


def decode_cases():
    rng = np.random.default_rng(6006)
    out = []
    for n, k, dim in ((1000, 64, 16), (777, 1, 7), (513, 256, 64), (40, 5, 3)):
        cb = rng.normal(0, 50, (k, dim))
        out.append(dict(idx=rng.integers(0, k, n).astype(np.uint32), cb=cb))
    return out


def distortion_cases():
    rng = np.random.default_rng(7007)
    out = []
    for n, dim, metric in ((1000, 16, "squared_euclidean"), (513, 7, "euclidean"), (3, 1, "squared_euclidean"),
                           (4096, 64, "squared_euclidean")):
        a = rng.normal(0, 30, (n, dim))
        out.append(dict(a=a, b=a + rng.normal(0, 3, (n, dim)), metric=metric))
    return out
