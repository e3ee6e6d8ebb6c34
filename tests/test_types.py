"""TrainingSet semantics (core.py:72-99) with the lazy float64 field of the
float32 path: same validation messages, a private immutable snapshot, the
float64 matrix equal to the exact widening, frozen attributes."""

import numpy as np
import pytest

from paper_0910_4711_b200 import TrainingSet, UsageError


def test_float32_snapshot_and_lazy_widening():
    x = np.random.default_rng(3).normal(size=(1000, 16)).astype(np.float32)
    ts = TrainingSet(x)
    assert (ts.m, ts.k) == (1000, 16)
    assert ts.__dict__["_f64"] is None  # nothing widened yet
    x[0, 0] = 1e9  # the caller's array is not the snapshot
    v = ts.vectors
    assert v.dtype == np.float64 and v[0, 0] != 1e9
    x[0, 0] = v[0, 0]
    assert np.array_equal(v, x.astype(np.float64))
    assert ts.vectors is v  # cached
    with pytest.raises(ValueError):
        v[0, 0] = 1.0
    with pytest.raises(AttributeError):
        ts.vectors = v


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_nonfinite_message_names_row_and_component(dtype):
    x = np.ones((5, 3), dtype=dtype)
    x[3, 2] = np.nan
    with pytest.raises(UsageError, match="training vector 3 component 2 is not finite"):
        TrainingSet(x)
    x[3, 2] = 1.0
    x[1, 0] = np.inf
    with pytest.raises(UsageError, match="training vector 1 component 0 is not finite"):
        TrainingSet(x)


@pytest.mark.parametrize("shape", [(0, 3), (3, 0)])
def test_empty_rejected(shape):
    for dtype in (np.float32, np.float64):
        with pytest.raises(UsageError, match="at least 1x1"):
            TrainingSet(np.ones(shape, dtype=dtype))


def test_float64_path_unchanged():
    x = np.random.default_rng(4).normal(size=(10, 4))
    ts = TrainingSet(x)
    assert ts.vectors is not x and np.array_equal(ts.vectors, x)
    assert not ts.vectors.flags.writeable
    assert TrainingSet([[1, 2], [3, 4]]).vectors.dtype == np.float64
