"""GPU sweep harness -- the reference's benchmark harness (``vqkit.bench``,
bench.py:1-156: codebook-size x worker-count sweeps, CSV output, the Amdahl
model) with the number of B200s in place of the number of threads
(the paper's Figure 3/4 protocol,
PAPER.md:646-659).

* ``run_sweep`` trains every (N, P) cell ``repeats`` times and keeps the
  minimum wall time, as bench.py:72-120 does.  P = 1 runs the design in this
  process (``parallel_lbg_train`` on one GPU); P > 1 spawns P processes, one
  per GPU, that run ``distributed.sharded_lbg_train`` over NCCL and report the
  slowest rank's time (barrier + device synchronise on both sides).
* ``write_bench_csv`` / ``speedup_report`` / ``amdahl_speedup`` keep the
  reference's CSV columns (``n,p,m,k,seconds,td,iterations``, p = GPUs) and
  report lines, so existing plots read the GPU sweep unchanged.
"""

from __future__ import annotations

import json
import os
import socket
import tempfile
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .core import SQUARED_EUCLIDEAN, LbgConfig, TrainingSet
from .errors import UsageError

BENCH_CSV_HEADER = "n,p,m,k,seconds,td,iterations"  # bench.py:15
DEFAULT_SIZES = (8, 16, 32, 64, 128)
DEFAULT_GPUS = (1, 2, 4, 8)
DEFAULT_REPEATS = 3
DEFAULT_SERIAL_FRACTION = 0.15


@dataclass(frozen=True)
class AmdahlParams:
    """Serial fraction S of the parallelized program and processor count n
    (bench.py:22-36)."""

    serial_fraction: float
    processors: int

    def __post_init__(self):
        if not 0.0 <= self.serial_fraction <= 1.0:
            raise UsageError(f"serial fraction must lie in [0, 1], got {self.serial_fraction}")
        if self.processors < 1:
            raise UsageError(f"processor count must be >= 1, got {self.processors}")


def amdahl_speedup(params: AmdahlParams) -> float:
    """speedup = 1 / (S + (1 - S) / n) (bench.py:39-43)."""
    s, n = params.serial_fraction, params.processors
    return 1.0 / (s + (1.0 - s) / n)


@dataclass(frozen=True)
class BenchRecord:
    """One sweep cell: a size-N codebook designed on P GPUs (``workers``
    keeps the reference's field name, bench.py:46-56)."""

    codebook_size: int
    workers: int
    vector_count: int
    dimension: int
    seconds: float
    td: float
    iterations: int


def synthetic_training_set(count: int, dimension: int, seed: int) -> TrainingSet:
    """Seeded uniform [0, 1) vectors (bench.py:59-62: same generator, same data)."""
    return TrainingSet(np.random.default_rng(seed).random((count, dimension)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, backend, data_path, cells, repeats, out_path, factory_spec, devices=0):
    """One rank of a P > 1 sweep column (spawned; one process per GPU, or --
    with fewer GPUs than ranks -- ranks sharing the visible GPUs over gloo,
    whose host-mediated collectives never make one rank's kernel wait on
    another's: the protocol and the results are the same, the times are not
    a scaling measurement)."""
    import importlib

    import torch
    import torch.distributed as dist

    from .distributed import sharded_lbg_train

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group(backend, init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    factory = None
    if factory_spec:
        mod, attr = factory_spec.split(":")
        factory = getattr(importlib.import_module(mod), attr)
    cuda = backend == "nccl" or devices > 0
    if cuda:
        os.environ["LOCAL_RANK"] = str(rank % max(1, devices) if devices else rank)
        torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    ts = TrainingSet(np.load(data_path))

    def sync():
        if cuda:
            torch.cuda.synchronize()

    # warm-up: first call per process pays module / context set-up
    sharded_lbg_train(TrainingSet(ts.vectors[: min(ts.m, 2048 * world)]),
                      LbgConfig(target_size=2, max_iterations_per_level=2, workers=world),
                      backend_factory=factory)
    results = []
    for cfg_kw in cells:
        config = LbgConfig(**cfg_kw)
        best, stats = None, None
        for _ in range(repeats):
            dist.barrier()
            sync()
            t0 = time.perf_counter()
            _, stats = sharded_lbg_train(ts, config, backend_factory=factory)
            sync()
            elapsed = torch.tensor([time.perf_counter() - t0], dtype=torch.float64,
                                   device="cuda" if cuda else "cpu")
            dist.all_reduce(elapsed, op=dist.ReduceOp.MAX)  # the slowest rank's time
            e = float(elapsed.item())
            best = e if best is None or e < best else best
        results.append({"seconds": best, "td": stats.total, "iterations": len(stats.history)})
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(results, f)
    dist.barrier()
    dist.destroy_process_group()


def run_sweep(ts: TrainingSet, sizes=DEFAULT_SIZES, gpu_counts=(1,), repeats: int = DEFAULT_REPEATS,
              epsilon: float = 1e-3, delta: float = 0.01, metric: str = SQUARED_EUCLIDEAN,
              max_iterations: int = 100, progress=None, backend: str = "nccl",
              backend_factory: str | None = None, thread_counts=None) -> list[BenchRecord]:
    """bench.run_sweep (bench.py:72-120) over GPU counts.  Every (N, P) cell
    is trained ``repeats`` times and the minimum wall time kept; only the
    design is timed.  ``backend``/``backend_factory`` ("module:callable" of a
    DeviceShard stand-in) exist so the P > 1 protocol runs on CPU with gloo."""
    if thread_counts is not None:  # the reference's keyword (bench.py:72-76): counts of GPUs here
        gpu_counts = tuple(thread_counts)
    if repeats < 1:
        raise UsageError(f"repeats must be >= 1, got {repeats}")
    for p in gpu_counts:
        if p < 1:
            raise UsageError(f"GPU count must be >= 1, got {p}")
    devices = 0
    if backend == "nccl":
        import torch

        have = torch.cuda.device_count()
        if have < 1:
            raise UsageError("the sweep needs a CUDA device")
        if max(gpu_counts) > have:
            # more ranks than GPUs: ranks share the GPUs over gloo (the
            # reference's thread counts stay meaningful as a protocol check)
            backend, devices = "gloo", have
    from .parallel import parallel_lbg_train

    cells = {}
    for gpus in gpu_counts:
        kws = [dict(target_size=s, epsilon=epsilon, delta=delta, workers=gpus,
                    max_iterations_per_level=max_iterations, distortion_metric=metric) for s in sizes]
        if gpus == 1 and backend_factory is None:
            parallel_lbg_train(TrainingSet(ts.vectors[: min(ts.m, 32)]),
                               LbgConfig(target_size=2, max_iterations_per_level=2))  # warm-up
            out = []
            for kw in kws:
                best, stats = None, None
                for _ in range(repeats):
                    t0 = time.perf_counter()
                    _, stats = parallel_lbg_train(ts, LbgConfig(**kw))
                    e = time.perf_counter() - t0
                    best = e if best is None or e < best else best
                out.append({"seconds": best, "td": stats.total, "iterations": len(stats.history)})
        else:
            import torch.multiprocessing as mp

            with tempfile.TemporaryDirectory() as tmp:
                data_path = os.path.join(tmp, "x.npy")
                x32 = ts.__dict__.get("_x32")
                np.save(data_path, x32 if x32 is not None else ts.vectors)
                out_path = os.path.join(tmp, "out.json")
                mp.spawn(_rank_main, args=(gpus, _free_port(), backend, data_path, kws, repeats,
                                           out_path, backend_factory, devices),
                         nprocs=gpus, join=True, start_method="spawn")
                with open(out_path) as f:
                    out = json.load(f)
        cells[gpus] = out
    records = []
    for size_i, size in enumerate(sizes):  # bench.py's cell order: size-major
        for gpus in gpu_counts:
            r = cells[gpus][size_i]
            rec = BenchRecord(codebook_size=size, workers=gpus, vector_count=ts.m, dimension=ts.k,
                              seconds=r["seconds"], td=r["td"], iterations=r["iterations"])
            records.append(rec)
            if progress is not None:
                progress(rec)
    return records


def write_bench_csv(records: list[BenchRecord], path, comment: str | None = None) -> None:
    """bench.write_bench_csv (bench.py:123-134): fixed columns, repr floats."""
    lines = [f"# {comment}"] if comment else []
    lines.append(BENCH_CSV_HEADER)
    for r in records:
        lines.append(f"{r.codebook_size},{r.workers},{r.vector_count},{r.dimension},"
                     f"{r.seconds!r},{r.td!r},{r.iterations}")
    Path(path).write_text("\n".join(lines) + "\n")


def speedup_report(records: list[BenchRecord],
                   serial_fraction: float = DEFAULT_SERIAL_FRACTION) -> list[str]:
    """bench.speedup_report (bench.py:137-156): measured speedup against the
    P = 1 cell of the same codebook size, Amdahl prediction alongside."""
    baselines = {r.codebook_size: r.seconds for r in records if r.workers == 1}
    lines = []
    for r in records:
        base = baselines.get(r.codebook_size)
        if base is None:
            continue
        measured = base / r.seconds if r.seconds > 0 else float("inf")
        predicted = amdahl_speedup(AmdahlParams(serial_fraction, r.workers))
        lines.append(f"N={r.codebook_size} P={r.workers}: measured speedup {measured:.2f}x, "
                     f"Amdahl prediction {predicted:.2f}x (serial fraction {serial_fraction:g})")
    return lines
