"""Device-drawn Gaussian-mixture training sets (the
generator half): every float bit of the rows vqb_open_gmm draws on the B200
equals the host restatement (oracle/vq_oracle.c vqo_gmm_rows), at the
oracle-friendly sizes and at cfg4's full 2^24 x 16; shards are slices of the
same set; and a design on device-drawn rows equals the oracle's design on the
restated rows (the reference's lbg_train, core.py:366-430)."""

import hashlib

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

vq = pytest.importorskip("paper_0910_4711_b200")
from paper_0910_4711_b200 import synthetic  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    from paper_0910_4711_b200 import _lib
    if _lib.device_count() < 1:
        pytest.fail("GPU tests need a CUDA device")


def _params(cfg):
    spec = synthetic.WORKLOADS[cfg]
    return spec, synthetic.mixture_params(np.random.default_rng(spec.seed), *synthetic._MIXTURES[cfg])


@pytest.mark.parametrize("cfg", ["cfg2", "cfg4", "cfg5"])
def test_device_rows_equal_host_restatement(cfg):
    spec, p = _params(cfg)
    n = 1 << 16
    ts, _ = synthetic.make_training_device(cfg, n)
    want = oracle.gmm_rows(p.means, p.sigmas, p.cum_weights, n, spec.seed)
    assert ts.vectors.dtype == np.float64
    got = ts._rows32()
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("dim", [1, 2, 3, 5, 8, 13, 64])
def test_device_rows_any_dimension(dim):
    """Partial Box-Muller groups (dim % 4 != 0) and very wide rows."""
    rng = np.random.default_rng(dim)
    p = synthetic.mixture_params(rng, dim, 37, 0.5, 3.0, dirichlet=dim % 2 == 1)
    n = 5000
    ts = synthetic.device_mixture(p, n, seed=0xDEADBEEF12345678)
    want = oracle.gmm_rows(p.means, p.sigmas, p.cum_weights, n, 0xDEADBEEF12345678)
    assert ts._rows32().tobytes() == want.tobytes()


def test_shards_are_slices_of_the_same_set():
    """Row g draws from counter g: shards [0, a) and [a, n) concatenate to the
    whole set, so a sharded design sees the rows a single device would."""
    spec, p = _params("cfg2")
    n, a = 1 << 15, 3 * 2048
    whole = synthetic.device_mixture(p, n, spec.seed)._rows32()
    s0 = synthetic.device_mixture(p, a, spec.seed, 0, n)._rows32()
    s1 = synthetic.device_mixture(p, n - a, spec.seed, a, n)._rows32()
    assert np.concatenate([s0, s1]).tobytes() == whole.tobytes()


def test_cfg4_full_size_bit_identical():
    """cfg4's 2^24 x 16 set (1 GiB) drawn on the device equals the host
    restatement bit for bit (SHA-256 of the float32 bytes)."""
    spec, p = _params("cfg4")
    ts, _ = synthetic.make_training_device("cfg4")
    got = hashlib.sha256(ts._rows32().tobytes()).hexdigest()
    want = hashlib.sha256(oracle.gmm_rows(p.means, p.sigmas, p.cum_weights, spec.n,
                                          spec.seed).tobytes()).hexdigest()
    assert got == want


def test_mixture_statistics():
    """The draws are the mixture they claim: per-component label frequencies
    follow the cumulative weights, standardised residuals are N(0, 1)."""
    rng = np.random.default_rng(11)
    p = synthetic.mixture_params(rng, 4, 8, 1.0, 2.0, dirichlet=True)
    n = 1 << 20
    x = synthetic.device_mixture(p, n, seed=99)._rows32().astype(np.float64)
    d = ((x[:, None, :] - p.means[None, :, :].astype(np.float64)) ** 2).sum(-1)
    lab = d.argmin(1)  # means are ~U(0,255)^4 apart, sigmas <= 2: unambiguous
    w = np.diff(np.concatenate([[0.0], p.cum_weights]))
    freq = np.bincount(lab, minlength=8) / n
    assert np.all(np.abs(freq - w) <= 5 * np.sqrt(w * (1 - w) / n) + 1e-6)
    z = (x - p.means[lab]) / p.sigmas[lab, None].astype(np.float64)
    assert abs(z.mean()) < 5e-3 and abs(z.var() - 1) < 5e-3
    assert abs(np.mean(z[:, 0] * z[:, 1])) < 5e-3  # Box-Muller pair partners uncorrelated


def test_design_on_device_rows_matches_oracle():
    spec, p = _params("cfg2")
    n = 1 << 15
    ts = synthetic.device_mixture(p, n, spec.seed)
    host = oracle.gmm_rows(p.means, p.sigmas, p.cum_weights, n, spec.seed)
    conf = vq.LbgConfig(target_size=64, epsilon=1e-3, delta=0.01)
    cb, stats = vq.lbg_train(ts, conf)
    ref = oracle.lbg_train(host.astype(np.float64), 64, epsilon=1e-3, delta=0.01,
                           workers=oracle.max_threads(), vectors32=host)
    assert [(h.codebook_size, h.iteration, h.empty_cells) for h in stats.history] == \
        [(s, i, e) for s, i, _, e in ref.history]
    np.testing.assert_allclose([h.td for h in stats.history], [h[2] for h in ref.history], rtol=1e-12)
    rel = np.abs(cb.codevectors - ref.codebook).max() / np.abs(ref.codebook).max()
    assert rel <= 1e-12


def test_encode_device_queries_matches_oracle():
    """cfg5-style: device-drawn queries encoded against a fixed codebook equal
    the oracle's encode of the restated queries."""
    spec, p = _params("cfg5")
    n = 1 << 16
    ts, _ = synthetic.make_training_device("cfg5", n)
    cb = np.random.default_rng(synthetic.CFG5_CODEBOOK_SEED).uniform(0, 255, (1024, 16))
    book = vq.Codebook(cb)
    got = vq.encode(ts, book)
    host = oracle.gmm_rows(p.means, p.sigmas, p.cum_weights, n, spec.seed)
    want = oracle.encode(host.astype(np.float64), cb, workers=oracle.max_threads())
    assert np.array_equal(np.asarray(got.indices), want)
