"""Multi-GPU host logic on CPU: world_size-2 gloo runs of the sharded design
driver (paper_0910_4711_b200/distributed.py: ShardPlan, run_sharded,
gather_rows, sharded_lbg_train).

The GPU backend (DeviceShard over libvqb200.so) is replaced by
``EmulatedShard``, a numpy restatement of the device pass protocol
(kernels.cu: epilogue -> packed int64 exchange buffer [K*L fixed-point sums |
K counts | distortion tile partials], finalize_kernel / apply_kernel state
machine) with the oracle doing the allocation.  The collectives are the real
torch.distributed calls over gloo, so what is tested is exactly the rank
protocol: one MAX allreduce for the fixed-point scale, one SUM allreduce of
the exchange buffer per pass, lockstep termination, the row all-gather for
per_worker -- and that the result is bit-identical for world sizes 1 and 2
and matches the reference's design (oracle) pass for pass.
"""

import math
import os
import socket
import sys

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TILE = 2048


def _fixed_plan(n_global: int, cmax: np.ndarray) -> tuple[np.ndarray, int]:
    """vqb200_internal.h fixed_plan: per-column shifts s_l = 61 - e_n - e_l
    (int64 high words of n rows cannot overflow) and the common low-word
    shift t = 62 - e_n."""
    e_n = 0
    while (1 << e_n) < n_global and e_n < 62:
        e_n += 1
    s = [max(-1020, min(960, 61 - e_n - (math.frexp(m)[1] if m > 0 else 0))) for m in cmax]
    return np.array(s, dtype=np.int64), 62 - e_n


def _lowbit(v: float) -> int:
    if v == 0.0:
        return 2**31 - 1
    m, e = math.frexp(abs(v))  # |v| = m 2^e, m in [0.5, 1)
    q = int(m * 2**53)
    return e - 53 + ((q & -q).bit_length() - 1)


class EmulatedShard:
    """numpy stand-in for distributed.DeviceShard (same method surface)."""

    def __init__(self, rows: np.ndarray, row_offset: int, n_global: int):
        import torch

        self.torch = torch
        self.x = np.ascontiguousarray(rows, dtype=np.float64)
        self.x32 = rows if rows.dtype == np.float32 else None
        self.n, self.dim = self.x.shape
        self.row_offset = row_offset
        self.n_global = n_global
        assert row_offset % TILE == 0
        self.ntiles = -(-n_global // TILE)

    # -- backend surface used by run_sharded ------------------------------
    def colstats(self) -> np.ndarray:
        cmax = np.max(np.abs(self.x), axis=0)
        clow = np.array([min(_lowbit(float(v)) for v in col) for col in self.x.T], dtype=np.float64)
        return np.concatenate([cmax, -clow])

    def tensor(self, values):
        return self.torch.tensor(values, dtype=self.torch.float64)

    def _plan(self, gstats) -> None:
        g = np.asarray(gstats, dtype=np.float64)
        self.shift, self.t = _fixed_plan(self.n_global, g[: self.dim])

    def _alloc_exchange(self) -> None:
        # [hi K*L | counts K | td tiles | lo K*L] (vqb200_internal.h Exchange)
        self.ex = self.torch.zeros(2 * self.kmax * self.dim + self.kmax + self.ntiles, dtype=self.torch.int64)

    def begin(self, config, gstats) -> None:
        self.cfg = config
        self.kmax = config.target_size
        self._plan(gstats)
        self._alloc_exchange()
        self.cb = np.zeros((self.kmax, self.dim))
        self.size, self.iteration, self.td_prev = 1, 1, math.inf
        self.done, self.mode_final = False, False
        self.hist, self.warn, self.total = [], [], 0.0
        self.pending_init = True
        self.dists = np.zeros(self.n)
        # initial column-sum pass: every row in cell 0 (epilogue with zero_cells)
        self._write_sums(np.zeros(self.n, dtype=np.int64), 1)

    def exchange(self):
        return self.ex

    def _split(self) -> tuple[np.ndarray, np.ndarray]:
        """kernels.cu split_fixed: x 2^s = hi + lo 2^-t, hi truncated toward 0."""
        v = self.x * np.exp2(self.shift.astype(np.float64))
        h = np.trunc(v)
        return h.astype(np.int64), ((v - h) * 2.0 ** self.t).astype(np.int64)

    def _write_sums(self, cells: np.ndarray, k: int) -> None:
        e = self.ex.numpy()
        kd = self.kmax * self.dim
        hi, lo = self._split()
        sums = np.zeros((k, self.dim), dtype=np.int64)
        los = np.zeros((k, self.dim), dtype=np.int64)
        np.add.at(sums, cells, hi)
        np.add.at(los, cells, lo)
        e[: k * self.dim] = sums.reshape(-1)
        e[kd: kd + k] = np.bincount(cells, minlength=k)
        lo0 = kd + self.kmax + self.ntiles
        e[lo0: lo0 + k * self.dim] = los.reshape(-1)

    def local(self) -> None:
        if self.done:
            return
        k = self.size
        metric = oracle.EUCLIDEAN if self.cfg.distortion_metric == "euclidean" else 0
        cells, dists = oracle.assign_all(self.x, self.cb[:k], metric)
        self.dists = dists
        e = self.ex.numpy()
        base = self.kmax * self.dim + self.kmax
        t0 = self.row_offset // TILE
        for t in range(-(-self.n // TILE)):
            s = 0.0
            for v in dists[t * TILE:(t + 1) * TILE]:
                s += v
            e[base + t0 + t] = np.float64(s).view(np.int64)
        self._write_sums(cells, k)

    def _set_action(self, update: bool, split: bool) -> None:
        e = self.ex.numpy()
        kd = self.kmax * self.dim
        k = self.size
        src = self.cb[:k].copy()
        if update:
            from fractions import Fraction

            counts = e[kd: kd + k]
            lo0 = kd + self.kmax + self.ntiles
            his = e[: k * self.dim].reshape(k, self.dim)
            los = e[lo0: lo0 + k * self.dim].reshape(k, self.dim)
            for c in range(k):
                if counts[c] == 0:
                    continue
                for l in range(self.dim):
                    # kernels.cu fixed_to_double: the exact sum rounded once
                    T = int(his[c, l]) * 2 ** self.t + int(los[c, l])
                    num = float(Fraction(T, 2 ** (int(self.shift[l]) + self.t)))
                    src[c, l] = np.float64(num) / np.float64(counts[c])
        if split:
            out = np.empty((2 * k, self.dim))
            out[0::2] = src + self.cfg.delta
            out[1::2] = src - self.cfg.delta
            self.cb[: 2 * k] = out
            self.size, self.iteration, self.td_prev = 2 * k, 1, math.inf
        else:
            self.cb[:k] = src

    def finalize(self) -> None:
        e = self.ex.numpy()
        base = self.kmax * self.dim + self.kmax
        if self.done:
            return
        if self.pending_init:
            self.pending_init = False
            if self.cfg.target_size <= 1:
                self.mode_final = True
                self._set_action(True, False)
            else:
                self._set_action(True, True)
            e[base: base + self.ntiles] = 0
            return
        k = self.size
        td = 0.0
        for t in range(self.ntiles):
            td += float(e[base + t: base + t + 1].view(np.float64)[0])
        e[base: base + self.ntiles] = 0
        if getattr(self, "lloyd", False):  # kModeLloydStep: update, done
            self._set_action(True, False)
            self.total, self.done = td, True
            return
        kd = self.kmax * self.dim
        empties = int(np.count_nonzero(e[kd: kd + k] == 0))
        if self.mode_final:
            self.total, self.done = td, True
            return
        p = self.td_prev
        conv = False if math.isinf(p) else (True if p == 0.0 else (p - td) / p <= self.cfg.epsilon)
        if conv:
            self.hist.append((k, self.iteration, td, 0))
            if k < self.cfg.target_size:
                self._set_action(False, True)
            else:
                self.total, self.done = td, True
            return
        self.hist.append((k, self.iteration, td, empties))
        self.td_prev = td
        self.iteration += 1
        if self.iteration > self.cfg.max_iterations_per_level:
            self.warn.append(k)
            if k < self.cfg.target_size:
                self._set_action(True, True)
            else:
                self._set_action(True, False)
                self.total, self.done = td, True
        else:
            self._set_action(True, False)

    def poll(self) -> bool:
        return self.done

    # -- fixed-size Lloyd passes (vqb_lloyd_*, distributed.sharded_lloyd)
    def lloyd_begin(self, codebook, gstats) -> None:
        import types

        cb = np.asarray(codebook, dtype=np.float64)
        self.cfg = types.SimpleNamespace(distortion_metric="squared_euclidean", delta=0.0)
        self.kmax = cb.shape[0]
        self._plan(gstats)
        self._alloc_exchange()
        self.cb = cb.copy()
        self.size, self.done, self.lloyd, self.pending_init = cb.shape[0], False, True, False

    def lloyd_local(self) -> None:
        self.done = False
        self.local()

    def lloyd_result(self):
        return self.cb.copy(), self.total

    def result(self):
        from paper_0910_4711_b200.core import LevelIteration, _max_iter_warning

        history = [LevelIteration(s, i, td, e) for s, i, td, e in self.hist]
        warnings = [_max_iter_warning(s, self.cfg.max_iterations_per_level) for s in self.warn]
        return self.cb[: self.size].copy(), history, warnings, self.total, self.dists


# ---------------------------------------------------------------------------
# worker processes
# ---------------------------------------------------------------------------

def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(name):
    rng = np.random.default_rng(11)
    if name == "gmm":
        means = rng.uniform(0, 255, (12, 4)).astype(np.float32)
        lab = rng.integers(0, 12, 5000)
        x = (means[lab] + rng.standard_normal((5000, 4)).astype(np.float32) * 6).astype(np.float32)
        cfg = dict(target_size=16, epsilon=1e-3, delta=0.01, workers=3)
    elif name == "tiny":  # fewer 2048-row tiles than ranks: replica fallback
        x = rng.random((300, 2))
        cfg = dict(target_size=4, epsilon=1e-3, delta=0.01, workers=5)
    else:  # guard exhaustion + euclidean, float64 input
        x = rng.random((4500, 3))
        cfg = dict(target_size=8, epsilon=0.0, delta=0.05, max_iterations_per_level=3,
                   distortion_metric="euclidean", workers=2)
    return x, cfg


def _worker(rank, world, port, name, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    for p in (ROOT, os.path.join(ROOT, "oracle")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch.distributed as dist

    import paper_0910_4711_b200 as vq
    from paper_0910_4711_b200 import distributed

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, cfg = _case(name)
        ts = vq.TrainingSet(x)
        cb, stats = distributed.sharded_lbg_train(ts, vq.LbgConfig(**cfg),
                                                  backend_factory=EmulatedShard)
        if rank == 0:
            np.savez(out_path, cb=cb.codevectors,
                     hist=np.array([(h.codebook_size, h.iteration, h.td, h.empty_cells)
                                    for h in stats.history]),
                     total=stats.total, per_worker=np.array(stats.per_worker),
                     nwarn=len(stats.warnings))
    finally:
        dist.destroy_process_group()


def _run(world, name, tmp_path):
    import torch.multiprocessing as mp

    out = str(tmp_path / f"{name}_w{world}.npz")
    mp.start_processes(_worker, args=(world, _free_port(), name, out), nprocs=world,
                       join=True, start_method="spawn")
    return np.load(out)


# ---------------------------------------------------------------------------
# tests
# ---------------------------------------------------------------------------

def test_shard_plan_tile_aligned_and_covering():
    from paper_0910_4711_b200.distributed import ShardPlan

    for n, world in [(5000, 2), (1 << 20, 8), (2049, 4), (100, 3), ((1 << 24) + 7, 8)]:
        plan = ShardPlan(n, world)
        cursor = 0
        for r in range(world):
            lo, hi = plan.bounds(r)
            assert lo == cursor and hi >= lo
            assert lo % TILE == 0 or lo == hi == n  # empty trailing shards only when tiles < world
            cursor = hi
        assert cursor == n
        tiles = [-(-(hi - lo) // TILE) for lo, hi in (plan.bounds(r) for r in range(world))]
        assert max(tiles) - min(tiles) <= 1


@pytest.mark.parametrize("name", ["gmm", "guard_euclidean", "tiny"])
def test_sharded_design_world2_matches_world1_and_reference(name, tmp_path):
    r1 = _run(1, name, tmp_path)
    r2 = _run(2, name, tmp_path)
    # world-size invariance: bit-identical codebook, history, total, per_worker
    for key in ("cb", "hist", "total", "per_worker", "nwarn"):
        assert r1[key].tobytes() == r2[key].tobytes(), key
    # and the reference's design (oracle), pass for pass
    x, cfg = _case(name)
    ref = oracle.lbg_train(np.asarray(x, dtype=np.float64), cfg["target_size"],
                           epsilon=cfg["epsilon"], delta=cfg["delta"], workers=cfg["workers"],
                           max_iterations_per_level=cfg.get("max_iterations_per_level", 100),
                           metric=cfg.get("distortion_metric", "squared_euclidean"))
    want = np.array(ref.history, dtype=np.float64)
    got = r2["hist"]
    assert got.shape == want.shape
    assert np.array_equal(got[:, [0, 1, 3]], want[:, [0, 1, 3]])
    np.testing.assert_allclose(got[:, 2], want[:, 2], rtol=1e-12)
    np.testing.assert_allclose(r2["cb"], ref.codebook, rtol=1e-12, atol=1e-12)
    assert int(r2["nwarn"]) == len(ref.warnings)
    np.testing.assert_allclose(r2["per_worker"], ref.per_worker, rtol=1e-12)


def _lloyd_worker(rank, world, port, out_path):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    from paper_0910_4711_b200 import distributed as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = _lloyd_data()
        plan = D.ShardPlan(x.shape[0], world)
        lo, hi = plan.bounds(rank)
        cb, td = D.sharded_lloyd(EmulatedShard(x[lo:hi], lo, x.shape[0]), x[:: 97][:64].astype(np.float64),
                                 passes=2, collective=world > 1)
        if rank == 0:
            np.savez(out_path, cb=cb, td=td)
    finally:
        dist.destroy_process_group()


def _lloyd_data():
    rng = np.random.default_rng(11)
    return rng.integers(0, 256, (3 * TILE + 123, 8)).astype(np.float32)


def test_sharded_lloyd_world2_matches_world1_and_oracle(tmp_path):
    """distributed.sharded_lloyd (the multi-GPU bench step): world 2 over gloo
    gives the world-1 codebook and distortion bit for bit, and the oracle's
    two Lloyd passes."""
    import torch.multiprocessing as mp

    outs = {}
    for world in (1, 2):
        out = str(tmp_path / f"l{world}.npz")
        mp.start_processes(_lloyd_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                           start_method="spawn")
        outs[world] = np.load(out)
    assert outs[1]["cb"].tobytes() == outs[2]["cb"].tobytes()
    assert float(outs[1]["td"]) == float(outs[2]["td"])
    x = _lloyd_data().astype(np.float64)
    cb = x[:: 97][:64].copy()
    for _ in range(2):
        cells, dists = oracle.assign_all(x, cb)
        td = oracle.sum_inorder(dists)
        cb, _ = oracle.update_codebook(x, cells, cb)
    assert np.array_equal(outs[2]["cb"], cb)  # pixel-valued rows: fixed-point sums are exact
    assert abs(float(outs[2]["td"]) - td) <= 1e-12 * td


def _per_worker_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_0910_4711_b200 import distributed as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 5 * TILE + 777
        d = np.random.default_rng(5).exponential(3.0, n)
        plan = D.ShardPlan(n, world)
        lo, hi = plan.bounds(rank)
        res = {w: D.sharded_per_worker(d[lo:hi], plan, rank, w, None) for w in (1, 2, 3, 7, 16)}
        if rank == 0:
            np.savez(out_path, **{str(w): np.array(v) for w, v in res.items()})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_per_worker_relay_is_the_inorder_sum(world, tmp_path):
    """per_worker from sharded distances without gathering them: chunks that
    span ranks are summed left to right by relaying the running sum, so
    every value equals sum_inorder over the chunk (parallel.py:321)."""
    import torch.multiprocessing as mp

    from paper_0910_4711_b200.parallel import _inorder, partition_training

    out = str(tmp_path / "pw.npz")
    mp.start_processes(_per_worker_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    r = np.load(out)
    n = 5 * TILE + 777
    d = np.random.default_rng(5).exponential(3.0, n)
    for w in (1, 2, 3, 7, 16):
        want = [_inorder(d[a:b]) for a, b in partition_training(n, w).ranges]
        assert r[str(w)].tolist() == want, w
