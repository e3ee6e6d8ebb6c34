"""float64 emulation of the tensor-core candidate pass's operands (the fp16
hi/lo split of centred rows and staged codevectors, kernels.cu /
assign_tc.cu): the exact value the MMA chain approximates, and the magnitude
sum that bounds its accumulation error.  Test helper only."""

import numpy as np


def session_mu(x32: np.ndarray) -> np.ndarray:
    """vqb_open's centre: FP64 ascending-row column sums of <= 4096 leading
    rows / m, rounded to FP32."""
    m = min(x32.shape[0], 4096)
    acc = np.cumsum(x32[:m].astype(np.float64), axis=0)[-1]
    return (acc / m).astype(np.float32)


def split16(v32: np.ndarray):
    hi = v32.astype(np.float16)
    lo = (v32 - hi.astype(np.float32)).astype(np.float16)
    return hi, lo


def expected_accumulators(x32, mu, cb64, ey, ew, kn):
    """(D_exact[rows, K], magnitude_sum[rows, K], v_exact[rows, K] * 2^(ey+ew))."""
    y = (x32.astype(np.float32) - mu).astype(np.float32)
    yh, yl = split16((y * np.float32(2.0 ** ey)).astype(np.float32))
    ct = (cb64 - mu.astype(np.float64)).astype(np.float32)
    w = (np.float32(-2.0) * ct).astype(np.float32)
    n = np.zeros(cb64.shape[0])
    for l in range(cb64.shape[1]):
        c = ct[:, l].astype(np.float64)
        n = n + c * c
    wh, wl = split16((w * np.float32(2.0 ** ew)).astype(np.float32))
    nv = n * 2.0 ** (ey + ew - kn)
    nh = nv.astype(np.float16)
    nl = (nv - nh.astype(np.float64)).astype(np.float16)
    f = lambda a: a.astype(np.float64)
    d = f(yh) @ f(wh).T + f(yh) @ f(wl).T + f(yl) @ f(wh).T + (2.0 ** kn) * (f(nh) + f(nl))[None, :]
    mag = np.abs(f(yh)) @ np.abs(f(wh)).T + np.abs(f(yh)) @ np.abs(f(wl)).T + \
        np.abs(f(yl)) @ np.abs(f(wh)).T + (2.0 ** kn) * np.abs(f(nh) + f(nl))[None, :]
    v = (y.astype(np.float64) @ w.astype(np.float64).T + n[None, :]) * 2.0 ** (ey + ew)
    return d, mag, v
