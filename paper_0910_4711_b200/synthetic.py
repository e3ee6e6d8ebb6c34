"""Seeded synthetic workloads for the five BASELINE.json configurations.

The reference ships no dataset: its only generator is uniform [0, 1)
(``bench.synthetic_training_set``, bench.py:59-62) and the paper's
2000-vector data is unspecified.  These generators pin
the prose of BASELINE.json ``configs``; every input
is generated once per process and the identical float32 array is handed to
the GPU path and to the CPU oracle.

Image blocks are vectorised exactly as ``storage.pixels_to_blocks``
(storage.py:281-293): row-major blocks, row-major pixels within a block.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "WorkloadSpec",
    "WORKLOADS",
    "blob_image",
    "image_blocks",
    "gaussian_mixture",
    "make_training",
    "make_encode_case",
    "MixtureParams",
    "mixture_params",
    "device_mixture",
    "make_training_device",
]


@dataclass(frozen=True)
class WorkloadSpec:
    name: str
    n: int
    dim: int
    target_size: int
    delta: float
    epsilon: float
    seed: int


WORKLOADS = {
    # cfg1: 512x512 image, 32 blobs, 4x4 blocks -> 16384 x 16, K=256
    "cfg1": WorkloadSpec("image4x4_512", 16384, 16, 256, 0.01, 1e-3, 1),
    # cfg2: 1024-component isotropic GMM, N=2^20, L=16, K=1024
    "cfg2": WorkloadSpec("gmm1024_n2e20_l16", 1 << 20, 16, 1024, 0.01, 1e-4, 2),
    # cfg3: 16 x 2048^2 images, 64 blobs each, 8x8 blocks -> 2^20 x 64, K=512
    "cfg3": WorkloadSpec("image8x8_16x2048", 1 << 20, 64, 512, 0.01, 1e-4, 3),
    # cfg4: 4096-component Dirichlet-weighted GMM, N=2^24, L=16, K=4096
    "cfg4": WorkloadSpec("gmm4096_n2e24_l16", 1 << 24, 16, 4096, 0.005, 1e-4, 4),
    # cfg5: encode 2^26 queries (cfg2 generator) against a fixed K=1024 codebook
    "cfg5": WorkloadSpec("encode_k1024_n2e26_l16", 1 << 26, 16, 1024, 0.0, 0.0, 51),
}

CFG5_CODEBOOK_SEED = 50


def blob_image(rng: np.random.Generator, height: int, width: int, blobs: int,
               noise_sigma: float = 8.0) -> np.ndarray:
    """Sum of ``blobs`` anisotropic rotated Gaussian blobs (centres uniform over
    the image, sigma_x, sigma_y ~ U(side/128, side/8), angle ~ U(0, pi),
    amplitude ~ U(0, 255)) plus N(0, noise_sigma^2) noise, clipped to [0, 255]
    and rounded to uint8.  Each blob is evaluated on its +-4 sigma window."""
    side = float(min(height, width))
    img = np.zeros((height, width), dtype=np.float32)
    params = []
    for _ in range(blobs):
        cy = rng.uniform(0, height)
        cx = rng.uniform(0, width)
        sx = rng.uniform(side / 128, side / 8)
        sy = rng.uniform(side / 128, side / 8)
        theta = rng.uniform(0, np.pi)
        amp = rng.uniform(0, 255)
        params.append((cy, cx, sx, sy, theta, amp))
    for cy, cx, sx, sy, theta, amp in params:
        r = 4.0 * max(sx, sy)
        y0, y1 = max(0, int(cy - r)), min(height, int(cy + r) + 1)
        x0, x1 = max(0, int(cx - r)), min(width, int(cx + r) + 1)
        if y1 <= y0 or x1 <= x0:
            continue
        yy = (np.arange(y0, y1, dtype=np.float32) - np.float32(cy))[:, None]
        xx = (np.arange(x0, x1, dtype=np.float32) - np.float32(cx))[None, :]
        c, s = np.float32(np.cos(theta)), np.float32(np.sin(theta))
        u = xx * c + yy * s
        v = yy * c - xx * s
        img[y0:y1, x0:x1] += np.float32(amp) * np.exp(
            -(u * u / np.float32(2 * sx * sx) + v * v / np.float32(2 * sy * sy)))
    img += rng.standard_normal((height, width), dtype=np.float32) * np.float32(noise_sigma)
    return np.rint(np.clip(img, 0, 255)).astype(np.uint8)


def image_blocks(pixels: np.ndarray, block: int) -> np.ndarray:
    """storage.pixels_to_blocks (storage.py:281-293) for images whose sides are
    multiples of ``block``; returns float32 (exact for 8-bit pixels)."""
    h, w = pixels.shape
    assert h % block == 0 and w % block == 0
    br, bc = h // block, w // block
    return (pixels.reshape(br, block, bc, block).swapaxes(1, 2)
            .reshape(br * bc, block * block).astype(np.float32))


def gaussian_mixture(rng: np.random.Generator, n: int, dim: int, components: int,
                     sigma_lo: float, sigma_hi: float, dirichlet: bool = False,
                     chunk: int = 1 << 22) -> np.ndarray:
    """Isotropic Gaussian mixture: means ~ U(0, 255)^dim, sigma ~ U(lo, hi),
    labels uniform (or Dirichlet(1)-weighted); float32 arithmetic."""
    means = rng.uniform(0, 255, (components, dim)).astype(np.float32)
    sig = rng.uniform(sigma_lo, sigma_hi, components).astype(np.float32)
    weights = rng.dirichlet(np.ones(components)) if dirichlet else None
    out = np.empty((n, dim), dtype=np.float32)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        if weights is None:
            labels = rng.integers(0, components, hi - lo)
        else:
            labels = rng.choice(components, hi - lo, p=weights)
        z = rng.standard_normal((hi - lo, dim), dtype=np.float32)
        np.multiply(z, sig[labels, None], out=z)
        np.add(z, means[labels], out=out[lo:hi])
    return out


def make_training(cfg: str, n: int | None = None) -> np.ndarray:
    """Float32 training matrix of BASELINE config ``cfg`` ('cfg1'..'cfg4').
    ``n`` truncates to the first n rows (parity tests at oracle-friendly size)."""
    spec = WORKLOADS[cfg]
    rng = np.random.default_rng(spec.seed)
    if cfg == "cfg1":
        x = image_blocks(blob_image(rng, 512, 512, 32), 4)
    elif cfg == "cfg2":
        x = gaussian_mixture(rng, spec.n if n is None else n, 16, 1024, 2.0, 20.0)
    elif cfg == "cfg3":
        images = 16 if n is None else max(1, -(-n // 65536))
        x = np.concatenate([image_blocks(blob_image(rng, 2048, 2048, 64), 8)
                            for _ in range(images)])
    elif cfg == "cfg4":
        x = gaussian_mixture(rng, spec.n if n is None else n, 16, 4096, 1.0, 16.0,
                             dirichlet=True)
    else:
        raise ValueError(f"no training set for {cfg}")
    return x if n is None else np.ascontiguousarray(x[:n])


def make_training_pixels(cfg: str, images: int = 16) -> np.ndarray:
    """The uint8 images behind make_training('cfg1') ([512, 512]) and
    make_training('cfg3') ([16, 2048, 2048]): same seeds, same draws, so
    pixels_to_blocks of these equals make_training(cfg); ``images`` < 16 gives
    the leading images of cfg3."""
    spec = WORKLOADS[cfg]
    rng = np.random.default_rng(spec.seed)
    if cfg == "cfg1":
        return blob_image(rng, 512, 512, 32)
    if cfg == "cfg3":
        return np.stack([blob_image(rng, 2048, 2048, 64) for _ in range(images)])
    raise ValueError(f"{cfg} is not an image workload")


def make_encode_case(n: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """cfg5: (codebook f32 [1024, 16] ~ U(0, 255), queries f32 [n, 16] from the
    cfg2 mixture generator with a separate seed)."""
    spec = WORKLOADS["cfg5"]
    cb = np.random.default_rng(CFG5_CODEBOOK_SEED).uniform(0, 255, (1024, 16)).astype(np.float32)
    q = gaussian_mixture(np.random.default_rng(spec.seed), spec.n if n is None else n,
                         16, 1024, 2.0, 20.0)
    return cb, q


# ---- device-drawn mixtures ----------------------------

@dataclass(frozen=True)
class MixtureParams:
    """Component parameters of an isotropic mixture: means [C, dim] f32,
    sigmas [C] f32, cumulative weights [C] f64 (None: uniform labels)."""
    means: np.ndarray
    sigmas: np.ndarray
    cum_weights: np.ndarray | None


def mixture_params(rng: np.random.Generator, dim: int, components: int, sigma_lo: float,
                   sigma_hi: float, dirichlet: bool = False) -> MixtureParams:
    """The component draws of ``gaussian_mixture`` (same rng calls, same
    order), so a device-drawn set samples the same mixture as the host one."""
    means = rng.uniform(0, 255, (components, dim)).astype(np.float32)
    sig = rng.uniform(sigma_lo, sigma_hi, components).astype(np.float32)
    cw = None
    if dirichlet:
        cw = np.minimum(np.cumsum(rng.dirichlet(np.ones(components))), 1.0)
        cw[-1] = 1.0
    return MixtureParams(means, sig, cw)


def device_mixture(params: MixtureParams, n: int, seed: int, row_offset: int = 0,
                   n_global: int | None = None, device: int | None = None):
    """A TrainingSet of ``n`` mixture rows drawn on the device (vqb_open_gmm):
    rows [row_offset, row_offset + n) of the ``n_global``-row set of ``seed``.
    Nothing but the component parameters crosses PCIe; the host ``vectors``
    field is downloaded only if something asks for it."""
    import ctypes

    from . import _lib
    from .core import TrainingSet, _Session, _device

    m = np.ascontiguousarray(params.means, dtype=np.float32)
    sg = np.ascontiguousarray(params.sigmas, dtype=np.float32)
    cw = None if params.cum_weights is None else np.ascontiguousarray(params.cum_weights, dtype=np.float64)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib().vqb_open_gmm(
        _lib.ptr(m), _lib.ptr(sg), _lib.ptr(cw), m.shape[0], n, m.shape[1], row_offset,
        row_offset + n if n_global is None else n_global, seed,
        _device() if device is None else device, ctypes.byref(h)))
    return TrainingSet._on_device(_Session.adopt(h, n, m.shape[1]))


_MIXTURES = {  # cfg -> (dim, components, sigma_lo, sigma_hi, dirichlet)
    "cfg2": (16, 1024, 2.0, 20.0, False),
    "cfg4": (16, 4096, 1.0, 16.0, True),
    "cfg5": (16, 1024, 2.0, 20.0, False),
}


def make_training_device(cfg: str, n: int | None = None, row_offset: int = 0,
                         n_global: int | None = None, device: int | None = None):
    """The device-drawn counterpart of ``make_training`` for the mixture
    configs (cfg2, cfg4; cfg5's queries): the same mixture components (same
    seed, same draws), rows from the counter-based device generator.  A shard
    [row_offset, row_offset + n) is the same slice of the same set on any
    number of devices.  Returns (TrainingSet, MixtureParams)."""
    if cfg not in _MIXTURES:
        raise ValueError(f"{cfg} is not a mixture workload")
    spec = WORKLOADS[cfg]
    params = mixture_params(np.random.default_rng(spec.seed), *_MIXTURES[cfg])
    rows = spec.n if n is None else n
    return device_mixture(params, rows, spec.seed, row_offset,
                          rows + row_offset if n_global is None else n_global, device), params
