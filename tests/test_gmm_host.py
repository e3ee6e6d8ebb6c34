"""Host side of the device mixture generator (no GPU): the restatement's
arithmetic (Philox4x32-10 known answers, series log / sin / cos against libm),
the component parameters equal the host generator's draws, and vqb_open_gmm
rejects bad parameters before touching a device."""

import ctypes
import math

import numpy as np
import pytest

import oracle
from paper_0910_4711_b200 import _lib, synthetic


def test_restatement_is_deterministic_and_sliceable():
    p = synthetic.mixture_params(np.random.default_rng(0), 6, 16, 1.0, 4.0, dirichlet=True)
    a = oracle.gmm_rows(p.means, p.sigmas, p.cum_weights, 4096, 7)
    b = oracle.gmm_rows(p.means, p.sigmas, p.cum_weights, 4096, 7)
    assert a.tobytes() == b.tobytes()
    tail = oracle.gmm_rows(p.means, p.sigmas, p.cum_weights, 1000, 7, row_offset=3096)
    assert tail.tobytes() == a[3096:].tobytes()
    assert oracle.gmm_rows(p.means, p.sigmas, p.cum_weights, 16, 8).tobytes() != a[:16].tobytes()


def test_standard_normal_draws():
    z = oracle.gmm_rows(np.zeros((1, 8), np.float32), np.ones(1, np.float32), None, 1 << 18, 3)
    z = z.astype(np.float64).ravel()
    assert abs(z.mean()) < 3e-3 and abs(z.var() - 1) < 5e-3
    # tails: P(|z| > 3) = 0.0027
    assert abs(np.mean(np.abs(z) > 3) - 0.0026998) < 4e-4


def test_series_match_libm():
    """The log and sin / cos series the generator uses stay within a few ulps
    of libm over (0, 1) in absolute terms: Box-Muller on them is the textbook transform."""
    u = (np.arange(1, 20001) - 0.5) / 20000
    # restated here in numpy with the same operation order
    b = u.view(np.uint64)
    e = ((b >> np.uint64(52)) & np.uint64(0x7FF)).astype(np.int64) - 1023
    m = ((b & np.uint64(0xFFFFFFFFFFFFF)) | np.uint64(0x3FF0000000000000)).view(np.float64)
    s = (m - 1.0) / (m + 1.0)
    s2 = s * s
    t = np.full_like(u, 1.0 / 27.0)
    for k in range(12, -1, -1):
        t = 1.0 / (2 * k + 1) + s2 * t
    lg = e * 0.6931471805599453 + 2.0 * s * t
    assert np.max(np.abs(lg - np.log(u))) < 4e-15  # absolute: log u -> 0 as u -> 1
    tt = u * 4.0
    q = tt.astype(np.int64)
    x = (tt - q) * 1.5707963267948966
    x2 = x * x
    ps = np.full_like(u, 1.0 / math.factorial(21))
    pc = np.full_like(u, 1.0 / math.factorial(20))
    for k in range(9, -1, -1):
        ps = 1.0 / math.factorial(2 * k + 1) - x2 * ps
        pc = 1.0 / math.factorial(2 * k) - x2 * pc
    assert np.max(np.abs(x * ps - np.sin(x))) < 5e-16
    assert np.max(np.abs(pc - np.cos(x))) < 5e-16


def test_mixture_params_are_the_host_generator_draws():
    """mixture_params makes the same rng calls, in the same order, as
    gaussian_mixture's component draws."""
    r1, r2 = np.random.default_rng(4), np.random.default_rng(4)
    p = synthetic.mixture_params(r1, 16, 64, 1.0, 16.0, dirichlet=True)
    means = r2.uniform(0, 255, (64, 16)).astype(np.float32)
    sig = r2.uniform(1.0, 16.0, 64).astype(np.float32)
    w = r2.dirichlet(np.ones(64))
    assert p.means.tobytes() == means.tobytes() and p.sigmas.tobytes() == sig.tobytes()
    assert p.cum_weights[-1] == 1.0 and np.all(np.diff(p.cum_weights) >= 0)
    np.testing.assert_allclose(np.diff(np.concatenate([[0], p.cum_weights])), w, atol=1e-15)
    assert r1.random() == r2.random()  # both streams advanced identically


def _open(means, sigmas, cw, comps, rows=16, dim=None):
    h = ctypes.c_void_p()
    dim = means.shape[1] if dim is None else dim
    return _lib.lib().vqb_open_gmm(_lib.ptr(means), _lib.ptr(sigmas), _lib.ptr(cw), comps, rows, dim, 0,
                                   rows, 1, 0, ctypes.byref(h))


def test_open_gmm_validates_before_the_device():
    m = np.zeros((3, 2), np.float32)
    s = np.ones(3, np.float32)
    assert _open(m, s, None, 0) == _lib.VQB_USAGE
    assert _open(m, -s, None, 3) == _lib.VQB_USAGE
    bad = m.copy()
    bad[1, 1] = np.nan
    assert _open(bad, s, None, 3) == _lib.VQB_USAGE
    assert _open(m, s, np.array([0.5, 0.4, 1.0]), 3) == _lib.VQB_USAGE   # decreasing
    assert _open(m, s, np.array([0.2, 0.4, 0.9]), 3) == _lib.VQB_USAGE   # does not end at 1
    assert b"cumulative" in _lib.lib().vqb_last_error()
    with pytest.raises(Exception):
        synthetic.make_training_device("cfg1")
