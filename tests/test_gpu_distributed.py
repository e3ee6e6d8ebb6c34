"""The sharded design on real hardware: two ranks (gloo, one process each)
drive DeviceShard sessions on the box's GPU through run_sharded -- the same
vqb_step_* loop and packed int64 exchange the NCCL path uses on an 8-GPU
node.  The collectives are host-mediated (gloo copies the device buffers),
so no kernel of one rank ever waits on the other.  The result must be the
single-device design, bit for bit, and the reference's schedule."""

import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data():
    sys.path.insert(0, ROOT)
    from paper_0910_4711_b200 import synthetic

    return synthetic.make_training("cfg2", n=(1 << 16) + 3000)  # ragged last shard


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    for p in (ROOT, os.path.join(ROOT, "oracle")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch
    import torch.distributed as dist

    import paper_0910_4711_b200 as vq

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = _data()
        cb, stats = vq.parallel_lbg_train(vq.TrainingSet(x),
                                          vq.LbgConfig(target_size=256, epsilon=1e-3, delta=0.01,
                                                       workers=3))
        if rank == 0:
            np.savez(out_path, cb=cb.codevectors,
                     hist=np.array([(h.codebook_size, h.iteration, h.td, h.empty_cells)
                                    for h in stats.history]),
                     total=stats.total, per_worker=np.array(stats.per_worker))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_design_matches_single_device(tmp_path):
    import torch.multiprocessing as mp

    import oracle
    import paper_0910_4711_b200 as vq

    out = str(tmp_path / "w2.npz")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True,
                       start_method="spawn")
    r2 = np.load(out)
    x = _data()
    cfg = vq.LbgConfig(target_size=256, epsilon=1e-3, delta=0.01, workers=3)
    cb1, st1 = vq.parallel_lbg_train(vq.TrainingSet(x), cfg)
    h1 = np.array([(h.codebook_size, h.iteration, h.td, h.empty_cells) for h in st1.history])
    # world-size invariance: identical bits
    assert r2["cb"].tobytes() == cb1.codevectors.tobytes()
    assert r2["hist"].tobytes() == h1.tobytes()
    assert float(r2["total"]) == st1.total
    np.testing.assert_array_equal(r2["per_worker"], np.array(st1.per_worker))
    # and the reference's pass schedule
    ref = oracle.lbg_train(x.astype(np.float64), 256, epsilon=1e-3, delta=0.01, workers=3)
    want = np.array(ref.history, dtype=np.float64)
    assert np.array_equal(h1[:, [0, 1, 3]], want[:, [0, 1, 3]])
    np.testing.assert_allclose(cb1.codevectors, ref.codebook, rtol=1e-12, atol=1e-12)


def _lloyd_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_0910_4711_b200 import distributed as D

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = _data()
        plan = D.ShardPlan(x.shape[0], world)
        lo, hi = plan.bounds(rank)
        shard = D.DeviceShard(np.ascontiguousarray(x[lo:hi]), lo, x.shape[0], 0)
        cb0 = np.ascontiguousarray(x[:: x.shape[0] // 256][:256].astype(np.float64))
        cb, td = D.sharded_lloyd(shard, cb0, passes=3)
        if rank == 0:
            np.savez(out_path, cb=cb, td=td)
    finally:
        dist.destroy_process_group()


def test_two_rank_lloyd_passes_match_single_device(tmp_path):
    """The multi-GPU bench step (vqb_lloyd_*: local pass, SUM allreduce of the
    exchange buffer, finalize) over two shards equals the same passes on one
    session holding every row, bit for bit, and the oracle's Lloyd passes."""
    import torch.multiprocessing as mp

    import oracle
    from paper_0910_4711_b200 import distributed as D

    out = str(tmp_path / "lloyd2.npz")
    mp.start_processes(_lloyd_worker, args=(2, _free_port(), out), nprocs=2, join=True,
                       start_method="spawn")
    r2 = np.load(out)
    x = _data()
    cb0 = np.ascontiguousarray(x[:: x.shape[0] // 256][:256].astype(np.float64))
    one = D.DeviceShard(x, 0, x.shape[0], 0)
    cb1, td1 = D.sharded_lloyd(one, cb0, passes=3, collective=False)
    assert r2["cb"].tobytes() == cb1.tobytes()
    assert float(r2["td"]) == td1
    cb = cb0
    x64 = x.astype(np.float64)
    for _ in range(3):
        cells, dists = oracle.assign_all(x64, cb)
        td = oracle.sum_inorder(dists)
        cb, _ = oracle.update_codebook(x64, cells, cb)
    np.testing.assert_allclose(cb1, cb, rtol=1e-12, atol=1e-12)
    assert abs(td1 - td) <= 1e-12 * td


def _nccl_one_rank(rank, port, out_path, graph):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), VQB_SHARD_GRAPH=graph)
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_0910_4711_b200 as vq
    from paper_0910_4711_b200.distributed import sharded_lbg_train

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        x = _data()
        cb, stats = sharded_lbg_train(vq.TrainingSet(x), vq.LbgConfig(target_size=64, epsilon=1e-3, delta=0.01))
        np.savez(out_path, cb=cb.codevectors, total=stats.total, passes=len(stats.history))
    finally:
        dist.destroy_process_group()


def test_nccl_graph_replayed_passes_match_plain_launches(tmp_path):
    """The sharded loop over NCCL with batches captured into a CUDA graph
    (kernels + allreduce) gives the bits of the plain per-pass launches."""
    import torch.multiprocessing as mp

    outs = []
    for graph in ("1", "0"):
        out = str(tmp_path / f"g{graph}.npz")
        mp.start_processes(_nccl_one_rank, args=(_free_port(), out, graph), nprocs=1, join=True,
                           start_method="spawn")
        outs.append(np.load(out))
    assert outs[0]["cb"].tobytes() == outs[1]["cb"].tobytes()
    assert float(outs[0]["total"]) == float(outs[1]["total"])
    assert int(outs[0]["passes"]) == int(outs[1]["passes"])


def test_programmatic_dependent_launch_is_transparent():
    """VQB_PDL=0 (plain stream order) and the default (programmatic dependent
    launches) design the same codebook bit for bit."""
    import subprocess

    code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_0910_4711_b200 as vq; "
            "from paper_0910_4711_b200 import synthetic; x = synthetic.make_training('cfg2', n=1 << 16); "
            "cb, st = vq.lbg_train(vq.TrainingSet(x), vq.LbgConfig(target_size=128, epsilon=1e-3)); "
            "sys.stdout.write(cb.codevectors.tobytes().hex()[:4096] + ' ' + repr(st.total))") % ROOT
    outs = []
    for pdl in ("1", "0"):
        env = dict(os.environ, VQB_PDL=pdl)
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                                   check=True, timeout=600).stdout)
    assert outs[0] == outs[1] and outs[0]


def _encode_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    for p in (ROOT, os.path.join(ROOT, "oracle")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch
    import torch.distributed as dist

    import paper_0910_4711_b200 as vq
    from paper_0910_4711_b200 import distributed as D

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = _data()
        rng = np.random.default_rng(77)
        cb = rng.uniform(0, 255, (1024, 16))
        stream = vq.encode(x, vq.Codebook(cb))          # the public API shards under a group
        idx, total = D.sharded_encode(x, cb, want_total=True)
        x64 = np.ascontiguousarray(x[:40000], dtype=np.float64) + 1e-9  # not float32-exact
        idx64, _ = D.sharded_encode(x64, cb)
        if rank == 0:
            np.savez(out_path, idx=stream.indices, idx2=idx, total=total, idx64=idx64)
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_encode_matches_single_device(tmp_path):
    """cfg5's sharding: every rank encodes its contiguous shard,
    the indices are all-gathered -- identical to one device and the oracle."""
    import torch.multiprocessing as mp

    import oracle
    import paper_0910_4711_b200 as vq

    out = str(tmp_path / "enc2.npz")
    mp.start_processes(_encode_worker, args=(2, _free_port(), out), nprocs=2, join=True,
                       start_method="spawn")
    r2 = np.load(out)
    x = _data()
    rng = np.random.default_rng(77)
    cb = rng.uniform(0, 255, (1024, 16))
    one = vq.encode(x, vq.Codebook(cb)).indices
    assert r2["idx"].dtype == np.uint32 and np.array_equal(r2["idx"], one)
    assert np.array_equal(r2["idx2"], one)
    cells, dists = oracle.assign_all(x.astype(np.float64), cb, workers=oracle.max_threads())
    assert np.array_equal(one, cells.astype(np.uint32))
    assert abs(float(r2["total"]) - float(np.sum(dists))) <= 1e-12 * float(np.sum(dists))
    x64 = np.ascontiguousarray(x[:40000], dtype=np.float64) + 1e-9
    c64, _ = oracle.assign_all(x64, cb)
    assert np.array_equal(r2["idx64"], c64.astype(np.uint32))
