"""Generate golden vectors by running the REFERENCE itself (vqkit, imported from
/root/reference/pkg/src in the build container).  The outputs are committed
under tests/golden/ so that parity tests never need /root/reference (which
does not exist on the GPU box).

Usage (build container only):
    python tests/golden/make_golden.py small        # kernel + small-design cases
    python tests/golden/make_golden.py cfg1 cfg2 cfg3 cfg5

Inputs are regenerated from seeds by the tests (tests/golden/cases.py and
paper_0910_4711_b200/synthetic.py); only reference OUTPUTS are stored.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import vqkit  # noqa: E402  (the reference)
from vqkit import _kernels  # noqa: E402

import cases  # noqa: E402
from paper_0910_4711_b200 import synthetic  # noqa: E402


def _save(name: str, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)", flush=True)


def small():
    out = {}
    for i, case in enumerate(cases.assign_cases()):
        x, cb, metric = case["x"], case["cb"], case["metric"]
        cells = np.empty(x.shape[0], dtype=np.int64)
        dists = np.empty(x.shape[0], dtype=np.float64)
        _kernels.assign_range(x, cb, 0, x.shape[0], metric, cells, dists)
        out[f"assign{i}_cells"] = cells
        out[f"assign{i}_dists"] = dists
        out[f"assign{i}_total"] = np.float64(_kernels.sum_inorder(dists))
    for i, case in enumerate(cases.update_cases()):
        x, cells, cb = case["x"], case["cells"], case["cb"]
        new = np.empty_like(cb)
        counts = np.zeros(cb.shape[0], dtype=np.int64)
        _kernels.update_rows(x, cells, cb, 0, 1, new, counts)
        out[f"update{i}_cb"] = new
        out[f"update{i}_counts"] = counts
    for i, case in enumerate(cases.design_cases()):
        ts = vqkit.TrainingSet(case["x"])
        cfg = vqkit.LbgConfig(**case["config"])
        cb, stats = vqkit.parallel_lbg_train(ts, cfg)
        out[f"design{i}_cb"] = cb.codevectors
        out[f"design{i}_hist"] = np.array([(h.codebook_size, h.iteration, h.td, h.empty_cells)
                                           for h in stats.history], dtype=np.float64).reshape(-1, 4)
        out[f"design{i}_total"] = np.float64(stats.total)
        out[f"design{i}_per_worker"] = np.array(stats.per_worker, dtype=np.float64)
        out[f"design{i}_nwarn"] = np.int64(len(stats.warnings))
    for i, case in enumerate(cases.encode_cases()):
        stream = vqkit.encode(case["x"], vqkit.Codebook(case["cb"]), workers=case["workers"])
        out[f"encode{i}_idx"] = stream.indices
    _save("small", **out)


class _Recorder:
    """Wraps vqkit.parallel._assign_phase (a module global looked up at call time
    by parallel_lbg_train, parallel.py:289) to record every allocation pass."""

    def __init__(self, keep_codebooks_upto: int):
        import vqkit.parallel as par
        self.par = par
        self.keep = keep_codebooks_upto
        self.counts, self.codebooks = [], {}
        self._real = par._assign_phase

    def __enter__(self):
        rec = self
        real = self._real

        def phase(vectors, rows, plan, code, cells, dists, executor):
            real(vectors, rows, plan, code, cells, dists, executor)
            p = len(rec.counts)
            rec.counts.append(np.bincount(cells, minlength=rows.shape[0]).astype(np.int32))
            if rows.shape[0] <= rec.keep:
                rec.codebooks[p] = rows.copy()

        self.par._assign_phase = phase
        return self

    def __exit__(self, *exc):
        self.par._assign_phase = self._real


def design(cfg: str, keep_codebooks_upto: int = 64):
    spec = synthetic.WORKLOADS[cfg]
    x = synthetic.make_training(cfg)
    ts = vqkit.TrainingSet(x)
    workers = os.cpu_count() or 1
    conf = vqkit.LbgConfig(target_size=spec.target_size, epsilon=spec.epsilon, delta=spec.delta,
                           workers=workers)
    t0 = time.perf_counter()
    with _Recorder(keep_codebooks_upto) as rec:
        cb, stats = vqkit.parallel_lbg_train(ts, conf)
    secs = time.perf_counter() - t0
    hist = np.array([(h.codebook_size, h.iteration, h.td, h.empty_cells) for h in stats.history],
                    dtype=np.float64)
    arrays = dict(cb=cb.codevectors, hist=hist, total=np.float64(stats.total),
                  seconds=np.float64(secs), workers=np.int64(workers), nwarn=np.int64(len(stats.warnings)),
                  x_sha256=np.bytes_(hashlib.sha256(x.tobytes()).hexdigest()))
    counts_flat = np.concatenate(rec.counts) if rec.counts else np.zeros(0, np.int32)
    arrays["pass_counts"] = counts_flat
    for p, c in rec.codebooks.items():
        arrays[f"pass{p}_cb"] = c
    _save(f"{cfg}_design", **arrays)


def encode_cfg5():
    cb, q = synthetic.make_encode_case()
    codebook = vqkit.Codebook(cb)
    t0 = time.perf_counter()
    workers = os.cpu_count() or 1
    stream = vqkit.encode(q, codebook, workers=workers)
    secs = time.perf_counter() - t0
    idx = stream.indices
    _, total = vqkit.assign_cells(q, codebook)
    _save("cfg5_encode", idx_sha256=np.bytes_(hashlib.sha256(idx.tobytes()).hexdigest()),
          bincount=np.bincount(idx, minlength=1024).astype(np.int64),
          head=idx[:65536].copy(), total=np.float64(total), seconds=np.float64(secs),
          workers=np.int64(workers),
          q_sha256=np.bytes_(hashlib.sha256(q.tobytes()).hexdigest()))


if __name__ == "__main__":
    for what in sys.argv[1:] or ["small"]:
        t = time.time()
        if what == "small":
            small()
        elif what == "cfg5":
            encode_cfg5()
        else:
            design(what)
        print(f"{what}: {time.time() - t:.1f}s", flush=True)
