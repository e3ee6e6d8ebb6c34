"""Multi-GPU LBG: one process per GPU, torch.distributed (NCCL) for the one
exchange per pass.

The reference's master/slave shared-memory scheme (parallel.py:256-329;
PAPER.md section 4: workers allocate disjoint chunks, the master integrates
tables and distortions) maps onto ranks as follows:

* rows are sharded into contiguous, tile-aligned ranges (``ShardPlan``; a tile
  is the 2048-row unit of the fixed distortion tree, so shard boundaries never
  split a tile and the result is bit-identical for every world size);
* every rank holds a codebook replica and runs allocation + epilogue on its
  shard (the C ABI's ``vqb_step_local``);
* the partial cell tables never move: each rank reduces them on the device
  into one packed int64 buffer [K*L fixed-point high words | K counts |
  distortion tile partials | K*L low words] (the two-word exact cell sums,
  vqb200_internal.h) and ONE ``all_reduce(SUM)`` over NVLink combines them --
  integer addition is exact, so the combined buffer is identical on every
  rank and for every world size;
* every rank then runs the same finalize (convergence test, centroids, split)
  on identical bits, so the "master" is implicit and no broadcast is needed.

The driver (``run_sharded``) is backend-agnostic so its collective logic is
tested on CPU with gloo (tests/test_distributed.py); ``DeviceShard`` is the
B200 backend over libvqb200.so.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib

TILE = 2048  # vqb200_internal.h kTdTile


def _split_stats(gstats: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """The MAX-reduced [colmax | -collow] vector back to the C ABI's arrays."""
    g = np.asarray(gstats, dtype=np.float64)
    dim = g.shape[0] // 2
    cmax = np.ascontiguousarray(g[:dim])
    clow = np.ascontiguousarray(-g[dim:]).astype(np.int32)
    return cmax, clow


def world_size() -> int:
    try:
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        return 1
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size()
    return 1


@dataclass(frozen=True)
class ShardPlan:
    """Contiguous tile-aligned row shards; the first (tiles mod world) ranks
    take one extra tile (the reference's partition rule, parallel.py:93-107,
    applied to 2048-row tiles)."""

    n: int
    world: int

    @property
    def tiles(self) -> int:
        return -(-self.n // TILE)

    def bounds(self, rank: int) -> tuple[int, int]:
        base, extra = divmod(self.tiles, self.world)
        t0 = rank * base + min(rank, extra)
        t1 = t0 + base + (1 if rank < extra else 0)
        return min(self.n, t0 * TILE), min(self.n, t1 * TILE)


class _CudaArray:
    """__cuda_array_interface__ view of a device buffer (zero-copy into torch)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {
            "shape": (count,), "typestr": "<i8", "data": (ptr, False), "version": 3}


class DeviceShard:
    """B200 backend: one vqb_session over this rank's rows."""

    def __init__(self, rows: np.ndarray, row_offset: int, n_global: int, device: int):
        from .core import _Session

        x32 = rows if rows.dtype == np.float32 else None
        x64 = None if x32 is not None else np.ascontiguousarray(rows, dtype=np.float64)
        self.s = _Session(x32, x64, device=device, row_offset=row_offset, n_global=n_global)
        self.device = device
        self.L = _lib.lib()
        import torch

        self.torch = torch
        # one stream for our kernels and the collectives between them (the
        # drivers below run the collectives under torch.cuda.stream(self.stream))
        self.stream = torch.cuda.Stream(device=device)
        _lib.check(self.L.vqb_set_stream(self.s.handle, ctypes.c_void_p(self.stream.cuda_stream)))
        self._ex = None

    def colstats(self) -> np.ndarray:
        """[max |x| per column | -(lowest set bit) per column] as float64: one
        MAX allreduce gives the global column stats of the fixed-point plan."""
        cmax, clow = self.s.colstats()
        return np.concatenate([cmax, -clow.astype(np.float64)])

    def tensor(self, values):
        return self.torch.tensor(values, dtype=self.torch.float64, device=f"cuda:{self.device}")

    def begin(self, config, gstats: np.ndarray) -> None:
        from .core import metric_code

        self.config = config
        cmax, clow = _split_stats(gstats)
        self._stats = (cmax, clow)  # alive for the call
        cfg = _lib.TrainConfig(config.target_size, config.epsilon, config.delta,
                               config.max_iterations_per_level,
                               metric_code(config.distortion_metric), 0,
                               cmax.ctypes.data, clow.ctypes.data)
        self._cfg = cfg
        _lib.check(self.L.vqb_step_begin(self.s.handle, ctypes.byref(cfg)))

    def exchange(self):
        if self._ex is None:
            p = ctypes.POINTER(ctypes.c_int64)()
            n = ctypes.c_int64()
            _lib.check(self.L.vqb_step_exchange(self.s.handle, ctypes.byref(p), ctypes.byref(n)))
            addr = ctypes.cast(p, ctypes.c_void_p).value
            self._ex = self.torch.as_tensor(_CudaArray(addr, int(n.value)),
                                            device=f"cuda:{self.device}")
        return self._ex

    def local(self) -> None:
        _lib.check(self.L.vqb_step_local(self.s.handle))

    # -- fixed-size Lloyd passes (vqb_lloyd_*): update_codebook after
    # assign_cells, sharded; the pass ends with the same exchange + finalize
    def lloyd_begin(self, codebook: np.ndarray, gstats: np.ndarray) -> None:
        cb = np.ascontiguousarray(codebook, dtype=np.float64)
        self._lloyd_k = cb.shape[0]
        cmax, clow = _split_stats(gstats)
        _lib.check(self.L.vqb_lloyd_begin(self.s.handle, _lib.ptr(cb), cb.shape[0], _lib.ptr(cmax),
                                          _lib.ptr(clow)))

    def lloyd_local(self) -> None:
        _lib.check(self.L.vqb_lloyd_local(self.s.handle))

    def lloyd_result(self) -> tuple[np.ndarray, float]:
        """(current codebook, distortion of the last pass)."""
        cb = np.empty((self._lloyd_k, self.s.dim), dtype=np.float64)
        summ = _lib.TrainSummary()
        hist = (_lib.LevelIterationC * 1)()
        warn = np.zeros(1, dtype=np.int64)
        _lib.check(self.L.vqb_step_result(self.s.handle, _lib.ptr(cb), hist, 1, _lib.ptr(warn), 1,
                                          None, ctypes.byref(summ)))
        return cb, float(summ.total)

    def finalize(self) -> None:
        _lib.check(self.L.vqb_step_finalize(self.s.handle))

    def poll(self) -> bool:
        d = ctypes.c_int()
        _lib.check(self.L.vqb_step_poll(self.s.handle, ctypes.byref(d)))
        return bool(d.value)

    def result(self):
        from .core import LevelIteration, _max_iter_warning

        config = self.config
        warn = np.zeros(64, dtype=np.int64)
        cb = np.empty((config.target_size, self.s.dim), dtype=np.float64)
        dists = np.empty(self.s.rows, dtype=np.float64)
        summ = _lib.TrainSummary()
        _lib.check(self.L.vqb_step_result(self.s.handle, _lib.ptr(cb), None, 0, _lib.ptr(warn), 64,
                                          _lib.ptr(dists), ctypes.byref(summ)))
        history = self.s.history(int(summ.n_hist))
        warnings = [_max_iter_warning(int(s), config.max_iterations_per_level)
                    for s in warn[: int(summ.n_warn)]]
        return cb[: int(summ.final_size)], history, warnings, float(summ.total), dists


def _capture_batch(backend, ex, batch: int):
    """One CUDA graph of ``batch`` passes -- our kernels and the NCCL
    allreduce between them -- replayed per batch, so the host issues one
    launch per batch instead of ~12 per pass (what bounds the small-codebook
    levels when the shards are small).  Every kernel reads its size / mode from
    the device state and passes after `done` exit at once, so the same graph
    serves every level, as in the single-GPU vqb_train.  NCCL + DeviceShard
    only (gloo collectives cannot be captured); VQB_SHARD_GRAPH=0 disables."""
    import os

    import torch
    import torch.distributed as dist

    if os.environ.get("VQB_SHARD_GRAPH", "1") == "0" or getattr(backend, "stream", None) is None:
        return None
    if dist.get_backend() != "nccl":
        return None
    backend.stream.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=backend.stream):
        for _ in range(batch):
            backend.local()
            dist.all_reduce(ex, op=dist.ReduceOp.SUM)
            backend.finalize()
    return g


def _on_stream(backend):
    """The backend's stream as torch's current stream (collectives, events and
    graph replays then order with its kernels); a no-op for CPU backends."""
    import contextlib

    stream = getattr(backend, "stream", None)
    if stream is None:
        return contextlib.nullcontext()
    import torch

    return torch.cuda.stream(stream)


def run_sharded(backend, config, batch: int = 4, collective: bool = True):
    with _on_stream(backend):
        return _run_sharded(backend, config, batch, collective)


def _run_sharded(backend, config, batch: int, collective: bool):
    """Drive the pass loop on every rank.  Collectives: one MAX allreduce of
    the column stats (the common two-word fixed-point plan), then per pass
    one SUM allreduce of the packed int64 exchange buffer.  Ranks stay in lockstep because every rank
    derives `done` from identical combined bits.  ``collective=False`` runs
    the same loop on one rank without any collective."""
    import torch.distributed as dist

    def all_reduce(t, op):
        if collective:
            dist.all_reduce(t, op=op)

    gstats = backend.tensor(backend.colstats())
    all_reduce(gstats, dist.ReduceOp.MAX)
    backend.begin(config, gstats.cpu().numpy())
    ex = backend.exchange()
    all_reduce(ex, dist.ReduceOp.SUM)
    backend.finalize()
    levels = max(1, int(math.log2(config.target_size)))
    limit = (levels + 1) * (config.max_iterations_per_level + 1) + 2 * batch
    passes = 0
    graph = _capture_batch(backend, ex, batch) if collective else None
    while True:
        if graph is not None:
            graph.replay()
        else:
            for _ in range(batch):
                backend.local()
                all_reduce(ex, dist.ReduceOp.SUM)
                backend.finalize()
        passes += batch
        if backend.poll():
            break
        if passes > limit:
            from .errors import InternalError

            raise InternalError(f"sharded training did not terminate after {passes} passes")
    return backend.result()


def sharded_lloyd(backend, codebook: np.ndarray, passes: int = 1, collective: bool = True,
                  on_pass=None):
    with _on_stream(backend):
        return _sharded_lloyd(backend, codebook, passes, collective, on_pass)


def _sharded_lloyd(backend, codebook: np.ndarray, passes: int, collective: bool, on_pass):
    """``passes`` Lloyd iterations at a fixed codebook size over all ranks:
    one MAX allreduce of the column stats (the common fixed-point plan), then per pass
    local assign + epilogue, ONE SUM allreduce of the packed int64 exchange
    buffer, finalize (the centroids of the combined sums, identical bits on
    every rank).  ``on_pass(i)`` runs after each pass is enqueued (timing)."""
    import torch.distributed as dist

    gstats = backend.tensor(backend.colstats())
    if collective:
        dist.all_reduce(gstats, op=dist.ReduceOp.MAX)
    backend.lloyd_begin(codebook, gstats.cpu().numpy())
    ex = backend.exchange()
    for i in range(passes):
        backend.lloyd_local()
        if collective:
            dist.all_reduce(ex, op=dist.ReduceOp.SUM)
        backend.finalize()
        if on_pass is not None:
            on_pass(i)
    return backend.lloyd_result()


def _local_device() -> int:
    """This rank's GPU: LOCAL_RANK when torchrun set it, else torch's current
    device (a caller that never called set_device still gets its own GPU)."""
    import os

    import torch

    lr = os.environ.get("LOCAL_RANK")
    dev = int(lr) if lr is not None else torch.cuda.current_device()
    torch.cuda.set_device(dev)
    return dev


def sharded_per_worker(dists: np.ndarray, plan: ShardPlan, rank: int, workers: int,
                       device: str | None) -> list[float]:
    """DistortionStats.per_worker (parallel.py:321: sum_inorder of each worker
    chunk's distances, chunks from partition_training) from sharded per-row
    distances WITHOUT gathering them: a chunk that spans ranks is summed left
    to right by relaying its running FP64 sum from rank to rank (one scalar
    send/recv per shard boundary inside a chunk), so every chunk sum is the
    reference's exact sequential sum.  One SUM allreduce of the `workers`
    values (each set by the rank holding the chunk's end) finishes it."""
    import torch
    import torch.distributed as dist

    from .parallel import partition_training

    a, b = plan.bounds(rank)
    vals = np.zeros(max(1, workers), dtype=np.float64)
    for w, (lo, hi) in enumerate(partition_training(plan.n, workers).ranges):
        s_lo, s_hi = max(lo, a), min(hi, b)
        if s_lo >= s_hi:
            continue
        carry = 0.0
        if lo < a:  # the chunk began on an earlier rank: continue its running sum
            t = torch.zeros(1, dtype=torch.float64, device=device)
            dist.recv(t, src=rank - 1)
            carry = float(t.item())
        piece = dists[s_lo - a: s_hi - a]
        # sequential: carry, carry + d0, ... (cumsum accumulates left to right)
        acc = float(np.cumsum(np.concatenate([[carry], piece]))[-1])
        if hi > b:
            dist.send(torch.tensor([acc], dtype=torch.float64, device=device), dst=rank + 1)
        else:
            vals[w] = acc
    t = torch.from_numpy(vals).to(device) if device else torch.from_numpy(vals)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(v) for v in t.cpu().numpy()[:workers]]


def sharded_encode(rows: np.ndarray, codebook: np.ndarray, want_total: bool = False):
    """codec.encode (codec.py:62-93) over every rank of the default process
    group: each rank encodes its contiguous tile-aligned shard of the rows
    (the reference's chunk fan-out, codec.py:79-87 / parallel.py:93-107, one
    GPU per chunk), the indices are all-gathered so every rank returns the
    full uint32 array, and the distortion (when asked for) is one FP64 SUM
    allreduce.  Every rank passes the same rows."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    n, dim = rows.shape
    plan = ShardPlan(n, world)
    if plan.tiles < world:
        plan = ShardPlan(n, 1)  # too few rows to shard: rank 0's answer everywhere
    lo, hi = plan.bounds(rank) if plan.world > 1 else (0, n)
    dev = _local_device()
    gdev = f"cuda:{dev}" if dist.get_backend() == "nccl" else None
    cb = np.ascontiguousarray(codebook, dtype=np.float64)
    part = np.ascontiguousarray(rows[lo:hi])
    idx = np.empty(hi - lo, dtype=np.uint32)
    total = ctypes.c_double(0.0)
    if part.dtype == np.float32:
        _lib.check(_lib.lib().vqb_encode_f32(_lib.ptr(part), part.shape[0], dim, _lib.ptr(cb), cb.shape[0],
                                             dev, _lib.ptr(idx), ctypes.byref(total) if want_total else None))
    else:
        from .core import _Session

        s = _Session(None, np.ascontiguousarray(part, dtype=np.float64), device=dev)
        _c, _d, tot = s.assign(cb, 0, want_dists=False)
        idx[:] = _c.astype(np.uint32)
        total.value = tot
    if plan.world == 1:
        return idx, total.value
    longest = max(b - a for a, b in (plan.bounds(r) for r in range(world)))
    buf = torch.zeros(longest, dtype=torch.int32, device=gdev)
    buf[: idx.shape[0]] = torch.from_numpy(idx.view(np.int32)).to(buf.device)
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    out = np.empty(n, dtype=np.uint32)
    for r in range(world):
        a, b = plan.bounds(r)
        out[a:b] = parts[r][: b - a].cpu().numpy().view(np.uint32)
    tot = torch.tensor([total.value], dtype=torch.float64, device=gdev)
    if want_total:
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    return out, float(tot.item())


def sharded_lbg_train(ts, config, backend_factory=None):
    """parallel_lbg_train over all ranks of the default process group."""
    import torch
    import torch.distributed as dist

    from .core import Codebook, DistortionStats
    from .parallel import _inorder, partition_training

    rank, world = dist.get_rank(), dist.get_world_size()
    plan = ShardPlan(ts.m, world)
    if plan.tiles < world:
        # fewer 2048-row tiles than ranks: some shard would be empty.  Every
        # rank designs the whole (small) set on its own device instead -- the
        # result is the same bits everywhere, no collective needed.
        plan = ShardPlan(ts.m, 1)
        world, rank = 1, 0
        from .core import _session_of

        if backend_factory is None:
            cb, history, warnings, total, dists, _summ = _session_of(ts).train(config)
            per_worker = [_inorder(dists[a:b])
                          for a, b in partition_training(ts.m, config.workers).ranges]
            return Codebook(cb), DistortionStats(per_worker=per_worker, total=total,
                                                 history=history, warnings=warnings,
                                                 vector_count=ts.m)
    lo, hi = plan.bounds(rank)
    x32 = ts.__dict__.get("_x32")
    rows = (x32 if x32 is not None else ts.vectors)[lo:hi]
    if backend_factory is None:
        device = _local_device()
        backend = DeviceShard(np.ascontiguousarray(rows), lo, ts.m, device)
        gdev = f"cuda:{device}"
    else:
        backend = backend_factory(rows, lo, ts.m)
        dev = getattr(backend, "device", None)  # a DeviceShard from a caller's cache
        gdev = f"cuda:{dev}" if dev is not None else None
    if plan.world == 1:  # replica fallback above: no collective
        cb, history, warnings, total, dists = run_sharded(backend, config, collective=False)
        all_dists = dists
        per_worker = [_inorder(all_dists[a:b]) for a, b in partition_training(ts.m, config.workers).ranges]
    else:
        cb, history, warnings, total, dists = run_sharded(backend, config)
        per_worker = sharded_per_worker(dists, plan, rank, config.workers,
                                        gdev if dist.get_backend() == "nccl" else None)
    stats = DistortionStats(per_worker=per_worker, total=total, history=history,
                            warnings=warnings, vector_count=ts.m)
    return Codebook(cb), stats
