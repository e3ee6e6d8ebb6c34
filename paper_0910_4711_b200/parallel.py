"""Data-parallel engine -- drop-in for the reference's ``vqkit.parallel``
(parallel.py:1-329).

The reference's master/slave scheme over shared-memory threads (contiguous
row chunks for allocation, round-robin codevector ownership for updation,
futures-join barriers; section 4) becomes, on B200:

* one device: the whole pass is a grid of CTAs over row tiles; the
  "integrate" step is an order-free int64 reduction plus a fixed-tree FP64
  distortion sum (kernels.cu epilogue / finalize).  ``workers`` keeps its
  reference meaning -- the chunking used for ``DistortionStats.per_worker``.
* several devices (one process per GPU, torch.distributed over NCCL): rows
  are sharded across ranks, every rank keeps a codebook replica, and each
  pass ends with ONE allreduce of the packed int64 exchange buffer
  (``distributed.py``).

Partition helpers keep the reference's exact semantics and error messages.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import (
    SQUARED_EUCLIDEAN,
    CellTable,
    Codebook,
    DistortionStats,
    LbgConfig,
    TrainingSet,
    _session_of,
    metric_code,
)
from .errors import InternalError, UsageError

# Test instrumentation hook kept for signature compatibility
# (parallel.py:38-42); the device engine has no worker threads to delay.
_worker_hook = None


@dataclass(frozen=True)
class ChunkPlan:
    """P contiguous, disjoint index ranges covering [0, M), sizes within 1
    (parallel.py:45-72)."""

    ranges: tuple[tuple[int, int], ...]

    def __post_init__(self):
        if not self.ranges:
            raise UsageError("chunk plan needs at least one range")
        cursor = 0
        sizes = []
        for lo, hi in self.ranges:
            if lo != cursor or hi < lo:
                raise UsageError(
                    f"chunk ranges must be contiguous from 0, got ({lo}, {hi}) at {cursor}"
                )
            sizes.append(hi - lo)
            cursor = hi
        if max(sizes) - min(sizes) > 1:
            raise UsageError(f"chunk sizes must differ by at most 1, got {sizes}")

    @property
    def workers(self) -> int:
        return len(self.ranges)

    @property
    def total(self) -> int:
        return self.ranges[-1][1]


@dataclass(frozen=True)
class UpdateAssignment:
    """Round-robin ownership: worker phi owns c iff c mod workers == phi
    (parallel.py:75-90)."""

    workers: int

    def __post_init__(self):
        if self.workers < 1:
            raise UsageError(f"worker count must be >= 1, got {self.workers}")

    def worker_for(self, index: int) -> int:
        return index % self.workers

    def rows_for(self, worker: int, size: int) -> range:
        return range(worker, size, self.workers)


def partition_training(m: int, workers: int) -> ChunkPlan:
    """parallel.partition_training (parallel.py:93-107)."""
    if m < 1:
        raise UsageError(f"vector count must be >= 1, got {m}")
    if workers < 1:
        raise UsageError(f"worker count must be >= 1, got {workers}")
    base, extra = divmod(m, workers)
    ranges = []
    cursor = 0
    for rho in range(workers):
        size = base + (1 if rho < extra else 0)
        ranges.append((cursor, cursor + size))
        cursor += size
    return ChunkPlan(tuple(ranges))


def _inorder(values: np.ndarray) -> float:
    """Strict left-to-right FP64 sum (sum_inorder, _kernels.py:92-98):
    np.cumsum accumulates sequentially."""
    return float(np.cumsum(values)[-1]) if values.size else 0.0


def parallel_assign(ts: TrainingSet, codebook: Codebook, plan: ChunkPlan,
                    metric: str = SQUARED_EUCLIDEAN) -> tuple[list[CellTable], list[float]]:
    """parallel.parallel_assign (parallel.py:157-191): per-chunk partial cell
    tables and chunk distortions (chunk order), from one device pass."""
    if plan.total != ts.m:
        raise UsageError(f"plan covers {plan.total} vectors, training set has {ts.m}")
    if ts.k != codebook.k:
        raise UsageError(
            f"dimension mismatch: training set has {ts.k} components, "
            f"codebook has {codebook.k}"
        )
    cells, dists, _ = _session_of(ts).assign(codebook.codevectors, metric_code(metric))
    partials = [CellTable(cells[lo:hi].copy(), codebook.size, start=lo) for lo, hi in plan.ranges]
    distortions = [_inorder(dists[lo:hi]) for lo, hi in plan.ranges]
    return partials, distortions


def integrate(partials: list[CellTable], distortions: list[float]) -> tuple[CellTable, float]:
    """parallel.integrate (parallel.py:194-224): ordered concatenation and an
    ascending-worker distortion sum, with the same coverage checks."""
    if not partials:
        raise UsageError("nothing to integrate: no partial tables")
    if len(partials) != len(distortions):
        raise UsageError(f"{len(partials)} partial tables but {len(distortions)} distortions")
    size = partials[0].codebook_size
    cursor = 0
    arrays = []
    for partial in partials:
        if partial.codebook_size != size:
            raise InternalError(
                f"partial tables disagree on codebook size: {partial.codebook_size} vs {size}"
            )
        if partial.start != cursor:
            raise InternalError(
                f"cell-table coverage broken: expected next chunk at {cursor}, "
                f"got one starting at {partial.start}"
            )
        arrays.append(partial.cells)
        cursor += len(partial)
    table = CellTable(np.concatenate(arrays), size, start=0)
    total = 0.0
    for d in distortions:
        total += float(d)
    return table, total


def parallel_update(ts: TrainingSet, table: CellTable, codebook: Codebook,
                    workers: int) -> tuple[Codebook, int]:
    """parallel.parallel_update (parallel.py:227-253): identical to the
    sequential update for every worker count (the device sums are
    order-free int64)."""
    if len(table) != ts.m or table.start != 0:
        raise UsageError(f"cell table must cover all {ts.m} training vectors from index 0")
    if table.codebook_size != codebook.size:
        raise UsageError(
            f"cell table was built for {table.codebook_size} codevectors, "
            f"codebook has {codebook.size}"
        )
    UpdateAssignment(workers)
    new, _, empty = _session_of(ts).update(table.cells, codebook.codevectors)
    return Codebook(new), empty


def parallel_lbg_train(ts: TrainingSet, config: LbgConfig) -> tuple[Codebook, DistortionStats]:
    """parallel.parallel_lbg_train (parallel.py:256-329).  With an initialised
    torch.distributed process group of size > 1 the rows are sharded across
    the ranks' GPUs (every rank passes the full TrainingSet and gets the same
    result); otherwise the design runs on one device."""
    from . import distributed

    if distributed.world_size() > 1:
        return distributed.sharded_lbg_train(ts, config)
    cb, history, warnings, total, dists, _summ = _session_of(ts).train(config)
    plan = partition_training(ts.m, config.workers)
    per_worker = [_inorder(dists[lo:hi]) for lo, hi in plan.ranges]
    stats = DistortionStats(per_worker=per_worker, total=total, history=history,
                            warnings=warnings, vector_count=ts.m)
    return Codebook(cb), stats
