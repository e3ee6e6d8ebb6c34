"""Kernel-surface drop-in for the reference's ``vqkit._kernels``
(pkg/src/vqkit/_kernels.py:1-98).

Same five functions, same argument meaning, same out-parameter convention
(the caller allocates, the kernel writes in place), backed by libvqb200.so
(sm_100a) through the C ABI of include/vqb200.h.  Every reference caller
looks these functions up on the module object at call time (core.py:244,
258, 271, 315-316, 338, 380, 392-393, 402, 421-422; parallel.py:114, 121,
190, 273, 290, 316, 321; codec.py:89, 154-155), so rebinding the attributes
of ``vqkit._kernels`` to these swaps the compute under the unchanged
reference engine.

This surface moves host buffers over PCIe on every call (it has to: the
reference passes host arrays).  The device-resident entry points
(``lbg_train``, ``encode`` ...) are the fast path; this one exists so the
reference's own engine and tests can run on the B200 unmodified.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

SQUARED_EUCLIDEAN = 0  # _kernels.py:14
EUCLIDEAN = 1          # _kernels.py:15


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def assign_range(vectors, codebook, start, stop, metric, out_cells, out_dists):
    """_kernels.assign_range (_kernels.py:18-36): rows [start, stop) of
    ``vectors`` -> nearest codevector (lowest index on ties) into
    out_cells[z] (int64) and its distance into out_dists[z] (FP64, sqrt'ed
    under EUCLIDEAN)."""
    v, cb = _f64(vectors), _f64(codebook)
    if out_cells.dtype != np.int64 or out_dists.dtype != np.float64:
        raise TypeError("out_cells must be int64 and out_dists float64")
    if not (out_cells.flags.c_contiguous and out_dists.flags.c_contiguous):
        raise TypeError("output buffers must be C-contiguous")
    _lib.check(_lib.lib().vqb_assign_range(_lib.ptr(v), v.shape[0], v.shape[1], _lib.ptr(cb),
                                           cb.shape[0], int(start), int(stop), int(metric),
                                           _lib.ptr(out_cells), _lib.ptr(out_dists)))


def update_rows(vectors, cells, old_codebook, worker, stride, out_codebook, out_counts):
    """_kernels.update_rows (_kernels.py:39-66): centroids of the codevector
    rows i with i % stride == worker; rows without members keep
    old_codebook[i].  Other rows of the outputs are left untouched."""
    v, cb = _f64(vectors), _f64(old_codebook)
    c = np.ascontiguousarray(cells, dtype=np.int64)
    if out_codebook.dtype != np.float64 or out_counts.dtype != np.int64:
        raise TypeError("out_codebook must be float64 and out_counts int64")
    _lib.check(_lib.lib().vqb_update_rows(_lib.ptr(v), v.shape[0], v.shape[1], _lib.ptr(c),
                                          _lib.ptr(cb), cb.shape[0], int(worker), int(stride),
                                          _lib.ptr(out_codebook), _lib.ptr(out_counts)))


def pair_distance(a, b, metric) -> float:
    """_kernels.pair_distance (_kernels.py:69-78)."""
    va, vb = _f64(a), _f64(b)
    out = ctypes.c_double()
    _lib.check(_lib.lib().vqb_pair_distance(_lib.ptr(va), _lib.ptr(vb), va.shape[0], int(metric),
                                            ctypes.byref(out)))
    return out.value


def column_sums(vectors) -> np.ndarray:
    """_kernels.column_sums (_kernels.py:81-89), ascending row order."""
    v = _f64(vectors)
    out = np.empty(v.shape[1], dtype=np.float64)
    _lib.check(_lib.lib().vqb_column_sums(_lib.ptr(v), v.shape[0], v.shape[1], _lib.ptr(out)))
    return out


def sum_inorder(values) -> float:
    """_kernels.sum_inorder (_kernels.py:92-98), strict left to right."""
    v = _f64(values)
    out = ctypes.c_double()
    _lib.check(_lib.lib().vqb_sum_inorder(_lib.ptr(v), v.shape[0], ctypes.byref(out)))
    return out.value


def install(module) -> None:
    """Rebind the five kernel attributes of a ``vqkit._kernels`` module object
    to the B200 implementations."""
    for name in ("assign_range", "update_rows", "pair_distance", "column_sums", "sum_inorder"):
        setattr(module, name, globals()[name])
