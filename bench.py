"""Benchmark of the B200 LBG hot path (BASELINE.json metric: G vector-codeword
distance evals/s per Lloyd iteration; codebook design wall time).

Headline (default, N=1): BASELINE configs[3] (cfg4, the largest config that
fits one B200) -- N = 2^24 float32 vectors, L = 16, from the seeded
4096-component Dirichlet-weighted Gaussian mixture (paper_0910_4711_b200/
synthetic.py); a step is ONE Lloyd iteration at the final level K = 4096
(assign over all rows + FP64 re-rank + exact distortion + exact cell sums +
centroid update), starting from the reference's own converged K=4096 codebook
(tests/golden/cfg4_design.npz, produced by the reference).  Evals per step =
N * K.  L2 is flushed (256 MiB write) between timed steps (the 1 GiB input is
larger than L2 anyway).

N > 1 (torchrun): STRONG scaling -- every rank holds a contiguous tile-aligned
shard of the same global 2^24-row set (distributed.ShardPlan); each pass ends
with one NCCL allreduce of the packed int64 exchange buffer; time = max over
ranks; value = N * K / that time.

Keys beyond the base contract:
  e2e           same iteration through the C ABI with HOST buffers from pinned
                memory (vqb_lloyd_step_f32: H2D of X + codebook, D2H of the
                new codebook + distortion); e2e_pageable: from a plain numpy array
  roofline      dominant kernel (assign_tc<16>): algorithmic 3L flops per
                eval / its CUDA-event time, against the measured tensor peak,
                with the ALU-pipe ceiling of its argmin epilogue and the FP32
                FFMA peak (the north star's denominator) beside it
  cpu_baseline  oracle/ (C + OpenMP restatement of the reference kernels) on a
                bounded row sample of the same iteration, all host cores
  design        one full cfg4 design (1 -> 4096, 338 passes in the reference):
                device-resident wall time and through lbg_train from numpy
  cfg2          the cfg2 Lloyd iteration (BASELINE configs[1]) and its design
--impl reference prints the CPU arm on the same config dict (the reference is
Python + numba and cannot travel to the GPU box: its arithmetic runs as the
oracle/ port).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "G vector·codeword distance evals/s per Lloyd iter"
UNIT = "G evals/s"


def _rank_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _golden_codebook():
    g = np.load(os.path.join(ROOT, "tests", "golden", "cfg2_design.npz"))
    return np.ascontiguousarray(g["cb"]), g


def _cpu_info():
    try:
        import psutil
        cores = psutil.cpu_count(logical=False) or os.cpu_count()
    except Exception:
        cores = os.cpu_count()
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return int(cores or 1), model


def _host_threads() -> int:
    """Every host thread this process may run on (torchrun exports
    OMP_NUM_THREADS=1, which would make the OpenMP default a single core; the
    oracle's parallel loops take an explicit thread count instead)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_iteration_rate(x: np.ndarray, cb: np.ndarray, target_s: float = 4.0, repeats: int = 3):
    """Oracle (reference arithmetic, OpenMP over all host cores) Lloyd
    iteration = parallel assign + in-order TD + round-robin update, on a
    bounded leading-row sample.  Returns (G evals/s, sample rows, threads, s)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    threads = _host_threads()
    k = cb.shape[0]

    def one(rows):
        xs = np.ascontiguousarray(x[:rows], dtype=np.float64)
        t0 = time.perf_counter()
        cells, dists = oracle.assign_all(xs, cb, workers=threads)
        oracle.sum_inorder(dists)
        oracle.update_all(xs, cells, cb, workers=threads)
        return time.perf_counter() - t0

    probe = min(x.shape[0], 8192)
    one(probe)  # warm
    t = one(probe)
    rows = int(min(x.shape[0], max(probe, probe * target_s / max(t, 1e-6))))
    best = min(one(rows) for _ in range(repeats))
    return rows * k / best / 1e9, rows, threads, best


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def _measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    except (OSError, ValueError):
        return {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def _roofline(achieved, evals, assign_ms, ffma_peak_tflops, traffic, n, clocks, k):
    """Roofline of the dominant kernel, assign_tc<16> (tcgen05 kind::f16 MMA
    chain into TMEM + top-2 epilogue).  achieved = ALGORITHMIC flops (3L = 48
    per vector-codeword eval) per launch / its CUDA-event time.
    The tensor pipe is not what binds it: the two-read epilogue spends per
    value half an FMNMX3 (chunk minimum) and an FSETP (band count) on the ALU
    pipe -- 2 lane-slots at 16 lanes/clk/SMSP for register operands
    (profiles/r01_microbench.json fmnmx_2reg) -- plus a predicated IADD, so
    `limiter` reports that ALU ceiling; the role profiler (VQB_TC_PROF) shows
    the epilogue warps busy 93 % and the MMA warp waiting on them 54 %."""
    peaks, src = _measured_peaks()
    tensor_peak = float(peaks.get("bf16_tflops", 1590.0))
    mhz = (clocks.summary().get("sm_mhz") if clocks else None) or 1965.0
    alu_ops = 2.0
    alu_ceiling = 148 * 4 * 16 / alu_ops * mhz * 1e6  # evals/s
    evals_per_s = evals / (assign_ms * 1e-3)
    return {
        "bound": "tensor", "kernel": "assign_tc<16>",
        "achieved": achieved, "peak": tensor_peak, "unit": "TFLOP/s", "frac": achieved / tensor_peak,
        "peak_source": f"{src} bf16_tflops (dense burst; kind::f16 runs at the bf16 rate)",
        "algorithmic": f"3L = 48 flops per vector-codeword eval, N*K = {n}*{k} evals per launch",
        "issued_mma_tflops": evals * 2 * (3 * 16 + 16) / (assign_ms * 1e-3) / 1e12,
        "traffic": traffic.get("bytes_per_launch") if traffic else None,
        "algorithmic_bytes": n * 16 * 4 + n * 4,
        "limiter": {"pipe": "ALU (minimum + band count over TMEM values)", "alu_ops_per_eval": alu_ops,
                    "ceiling_g_evals_per_s": alu_ceiling / 1e9,
                    "frac": evals_per_s / alu_ceiling},
        "vs_fp32_ffma_peak": {"peak_tflops": ffma_peak_tflops, "frac": achieved / ffma_peak_tflops,
                              "peak_source": "measured FFMA microbenchmark (vqb_pipe_microbench)"},
    }


def _load_traffic(name):
    """DRAM bytes per launch of assign_tc<16> from the committed ncu --set full
    capture of this workload (profiles/assign_traffic_<cfg>.json)."""
    path = os.path.join(ROOT, "profiles", f"assign_traffic_{name}.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


LLOYD_WORKLOADS = ("cfg4", "cfg2")  # the Lloyd-iteration lines; cfg4 is the headline (largest 1-GPU config)


def _lloyd_case(name):
    """(spec, reference's converged codebook, golden npz) of a Lloyd-line workload."""
    from paper_0910_4711_b200 import synthetic

    g = np.load(os.path.join(ROOT, "tests", "golden", f"{name}_design.npz"))
    return synthetic.WORKLOADS[name], np.ascontiguousarray(g["cb"]), g


def _lloyd_config(name, n, k, world):
    """The `config` dict of a Lloyd-iteration line -- identical in both arms
    (bench.py --impl reference prints the same dict)."""
    from paper_0910_4711_b200 import synthetic

    spec = synthetic.WORKLOADS[name]
    return {"workload": f"{name}: {spec.name} N=2^{int(np.log2(n))} L=16, one Lloyd iteration at K={k} "
                        f"(reference's converged codebook)",
            "rows": n, "codebook": k, "dim": 16,
            "parallelism": f"dp{world}" if world > 1 else "single",
            "sharding": "contiguous tile-aligned row shards of the same global set (strong scaling)",
            "l2": "flushed (256 MiB write) between timed steps"}


def _cpu_lloyd(x, cb, target_s, warmup, steps):
    """Oracle (reference arithmetic, OpenMP over every host thread) Lloyd
    iteration on a bounded leading-row sample: parallel assign + in-order TD
    + update.  Returns (G evals/s, rows, threads, mean s per step)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    rate, rows, threads, _ = cpu_iteration_rate(x, cb, target_s=target_s, repeats=1)
    xs = np.ascontiguousarray(x[:rows], dtype=np.float64)
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        cells, dists = oracle.assign_all(xs, cb, workers=threads)
        oracle.sum_inorder(dists)
        oracle.update_all(xs, cells, cb, workers=threads)
        if i >= warmup:
            times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    return rows * cb.shape[0] / t / 1e9, rows, threads, t


def run_reference(args):
    """The CPU arm: the reference's own arithmetic (oracle/ C + OpenMP port of
    vqkit._kernels) on the SAME workload/config as the GPU arm, each step a
    bounded row sample of it.  Under torchrun only rank 0 runs."""
    rank, world, _ = _rank_env()
    if rank != 0:
        return 0
    from paper_0910_4711_b200 import synthetic

    name = args.workload if args.workload in LLOYD_WORKLOADS else "cfg4"
    spec, cb, _ = _lloyd_case(name)
    x = synthetic.make_training(name)
    cores, model = _cpu_info()
    steps = max(1, min(args.steps, 5))  # a bounded sample per step: the run stays within minutes
    value, rows, threads, t = _cpu_lloyd(x, cb, 2.0, min(args.warmup, 1), steps)
    sample = (f"{rows} leading rows of {name} x K={cb.shape[0]} (reference's converged codebook): "
              f"assign + in-order TD + update per step, {steps} steps")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": world, "steps": steps, "warmup": min(args.warmup, 1),
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _lloyd_config(name, x.shape[0], cb.shape[0], world),
        "cpu_model": model, "rows_sampled": rows,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _e2e_time(L, xh, cb, K, local_rank, flush, args, torch) -> float:
    """Mean seconds of one Lloyd iteration through vqb_lloyd_step_f32 (the C
    ABI with host buffers: H2D of this rank's rows + the codebook, D2H of the
    new codebook and distortion).  xh pinned (torch pin_memory, pinned at
    start-up: freshly pinned pages DMA at ~half rate for about a second,
    tools/e2e_probe3.py) or pageable numpy."""
    from paper_0910_4711_b200 import _lib

    new_cb = np.empty_like(cb)
    td = ctypes.c_double()
    empty = ctypes.c_int64()
    n = xh.shape[0]

    def e2e_step():
        # the step's result is the new codebook + distortion (what the next
        # Lloyd pass consumes); the cell table stays on the device
        _lib.check(L.vqb_lloyd_step_f32(_lib.ptr(xh), n, 16, _lib.ptr(cb), K, local_rank,
                                        _lib.ptr(new_cb), None, ctypes.byref(td), ctypes.byref(empty)))

    for _ in range(max(1, min(args.warmup, 2))):
        e2e_step()
    times = []
    for _ in range(max(1, min(args.steps, 10))):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()
        times.append(time.perf_counter() - t0)
    return sum(times) / len(times)


def _timed_lloyd(shard, cb, world, dist, flush, warmup, steps, torch):
    """Lloyd passes of distributed.sharded_lloyd on one rank: local assign +
    re-rank + distortion + cell sums, ONE SUM allreduce of the packed int64
    exchange buffer over NCCL (world > 1), finalize; CUDA events on the stream
    all of it runs on.  Returns the per-step ms of this rank."""
    with torch.cuda.stream(shard.stream):  # our kernels, NCCL and the events on one stream
        gstats = shard.tensor(shard.colstats())
        if world > 1:
            dist.all_reduce(gstats, op=dist.ReduceOp.MAX)
        shard.lloyd_begin(cb, gstats.cpu().numpy())
        ex = shard.exchange()

        def pass_():
            shard.lloyd_local()
            if world > 1:
                dist.all_reduce(ex, op=dist.ReduceOp.SUM)
            shard.finalize()

        for _ in range(warmup):
            flush.zero_()
            pass_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = []
        for _ in range(steps):
            flush.zero_()
            torch.cuda.synchronize()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record()
            pass_()
            ev1.record()
            torch.cuda.synchronize()
            ms.append(ev0.elapsed_time(ev1))
        torch.cuda.synchronize()
    return ms


def _design_entry(sess, x, conf, golden, vq, torch, e2e_runs=2):
    """One full design: device-resident wall time (vqb_train on the resident
    session) and through lbg_train from a numpy float32 matrix, with the
    reference schedule check."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dcb, hist, warns, total, _d, summ = sess.train(conf)
    design_s = time.perf_counter() - t0
    walls = []
    for _ in range(e2e_runs):  # the first call also pays one-time staging / module setup
        t0 = time.perf_counter()
        vq.lbg_train(vq.TrainingSet(x), conf)  # host buffer -> device -> host
        walls.append(time.perf_counter() - t0)
    ghist = golden["hist"]
    return {
        "wall_s": design_s, "e2e_wall_s": min(walls[1:] if len(walls) > 1 else walls),
        "passes": int(summ.passes), "evals": int(summ.evals),
        "g_evals_per_s": summ.evals / design_s / 1e9,
        "flagged_rows": int(summ.flagged_rows), "flagged_full_scan_rows": int(summ.flagged_full),
        "sums_exact": int(summ.sums_exact), "sums_ref_exact": int(summ.ref_exact),
        "reference_passes": int(ghist.shape[0]),
        "schedule_matches_reference": bool(
            len(hist) == ghist.shape[0] and all(
                (h.codebook_size, h.iteration, h.empty_cells) == (int(g[0]), int(g[1]), int(g[3]))
                for h, g in zip(hist, ghist))),
        "total_rel_err_vs_reference": abs(total - float(golden["total"])) / float(golden["total"]),
        "codebook_max_rel_err_vs_reference": float(np.max(np.abs(dcb - golden["cb"]) /
                                                          np.maximum(np.abs(golden["cb"]), 1e-300))),
        "reference_wall_s": float(golden["seconds"]),
        "reference_workers": int(golden["workers"]) if "workers" in golden.files else None,
    }


def run_b200(args):
    """The headline Lloyd-iteration line (default cfg4; --workload cfg2 for
    the cfg2 line).  N > 1: strong scaling -- every rank holds a contiguous
    tile-aligned shard (distributed.ShardPlan) of the same global set."""
    rank, world, local_rank = _rank_env()
    import torch

    import paper_0910_4711_b200 as vq
    from paper_0910_4711_b200 import _lib, synthetic
    from paper_0910_4711_b200 import distributed as D
    from paper_0910_4711_b200.core import _Session

    name = args.workload if args.workload in LLOYD_WORKLOADS else "cfg4"
    torch.cuda.set_device(local_rank)
    L = _lib.lib()
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))

    spec, cb, golden = _lloyd_case(name)
    K = cb.shape[0]
    x = synthetic.make_training(name)  # every rank: the same global set
    n = x.shape[0]
    plan = D.ShardPlan(n, world)
    lo, hi = plan.bounds(rank)
    xs = np.ascontiguousarray(x[lo:hi])
    n_local = xs.shape[0]
    xp_t = torch.from_numpy(xs).pin_memory()  # e2e input (this rank's shard), pinned early
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local_rank}")

    # ---- peak: measured FFMA throughput (lane FMA/s -> FLOP/s)
    ops, sec = ctypes.c_double(), ctypes.c_double()
    _lib.check(L.vqb_pipe_microbench(0, 4, 4000, ctypes.byref(ops), ctypes.byref(sec)))
    ffma_peak_tflops = 2 * ops.value / 1e12

    # ---- per-kernel segments of this rank's local pass (roofline diagnostic)
    sess = _Session(xs, None, device=local_rank, row_offset=lo, n_global=n)
    segs = (ctypes.c_double * 5)()
    flagged = ctypes.c_int64()

    def seg_step():
        _lib.check(L.vqb_bench_iteration(sess.handle, _lib.ptr(cb), K, 1, segs, ctypes.byref(flagged)))
        return list(segs)

    clocks = ClockSampler(local_rank).__enter__()
    for _ in range(args.warmup):
        flush.zero_()
        seg_step()
    seg_hist = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        seg_hist.append(seg_step())
    seg = [sum(s[k] for s in seg_hist) / len(seg_hist) for k in range(5)]

    # ---- the timed step: whole Lloyd passes of the (multi-GPU) loop
    shard = D.DeviceShard(xs, lo, n, local_rank)
    ms_steps = _timed_lloyd(shard, cb, world, dist, flush, args.warmup, args.steps, torch)
    ms_step = sum(ms_steps) / len(ms_steps)
    if world > 1:
        t = torch.tensor([ms_step], dtype=torch.float64, device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
        dist.barrier()
    evals = n * K
    value = evals / (ms_step * 1e-3) / 1e9
    assign_ms = seg[1]
    achieved = 3 * 16 * n_local * K / (assign_ms * 1e-3) / 1e12
    traffic = _load_traffic(name)

    if getattr(args, "profile_steps", False):
        clocks.__exit__(None, None, None)
        if rank == 0:
            print(json.dumps({"profile_steps": args.steps, "ms_per_step": ms_step,
                              "segments_ms": seg}), flush=True)
        return 0
    # ---- e2e on every rank at once (each uploads its own shard over its own
    # PCIe link): the slowest rank's time is the job's
    e2e_s = _e2e_time(L, xp_t.numpy(), cb, K, local_rank, flush, args, torch)
    e2e_pg_s = _e2e_time(L, xs, cb, K, local_rank, flush, args, torch)  # pageable numpy rows
    if world > 1:
        t = torch.tensor([e2e_s, e2e_pg_s], dtype=torch.float64, device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s, e2e_pg_s = (float(v) for v in t.tolist())
    clocks.__exit__(None, None, None)  # every rank: the sampler is a child process
    c = clocks.summary()
    if rank == 0:
        design, second = {}, {}
        if world == 1:
            del shard
            conf = vq.LbgConfig(target_size=spec.target_size, epsilon=spec.epsilon, delta=spec.delta)
            design = _design_entry(sess, x, conf, golden, vq, torch, e2e_runs=1 if name == "cfg4" else 3)
            if name == "cfg4":
                # the cfg2 line (BASELINE configs[1]) beside the headline
                del sess
                torch.cuda.empty_cache()
                s2, cb2, g2 = _lloyd_case("cfg2")
                x2 = synthetic.make_training("cfg2")
                sh2 = D.DeviceShard(x2, 0, x2.shape[0], local_rank)
                ms2 = _timed_lloyd(sh2, cb2, 1, None, flush, args.warmup, args.steps, torch)
                del sh2
                sess2 = _Session(x2, None, device=local_rank)
                conf2 = vq.LbgConfig(target_size=s2.target_size, epsilon=s2.epsilon, delta=s2.delta)
                m2 = sum(ms2) / len(ms2)
                second = {"cfg2": {"config": _lloyd_config("cfg2", x2.shape[0], cb2.shape[0], 1),
                                   "value": x2.shape[0] * cb2.shape[0] / (m2 * 1e-3) / 1e9, "unit": UNIT,
                                   "ms_per_step": m2,
                                   "design": _design_entry(sess2, x2, conf2, g2, vq, torch)}}

        # ---- CPU baseline: oracle on a bounded sample, all host cores
        cpu_rate, rows, threads, secs = cpu_iteration_rate(x, cb, target_s=4.0)
        cores, model = _cpu_info()
        # per step: reset, assign_fast + assign_small + assign_tc (two of them
        # exit at once), TC shortlist + FP32 shortlist + exact re-rank, td_tiles
        # (+ low-word clear) + sums_red + sums (one exits) + reduce_partials,
        # finalize + apply (profiles/r02_launch_summary_cfg4_step.txt)
        launches_per_step = 13
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32+f64", "data": "synthetic",
            "config": _lloyd_config(name, n, K, world),
            "step": ("Lloyd pass: local assign + re-rank + distortion + cell sums, "
                     + ("NCCL allreduce of the packed int64 exchange buffer, " if world > 1 else "")
                     + "finalize (distributed.sharded_lloyd); CUDA events around each whole pass"),
            "segments_ms": {"stage": seg[0], "assign": seg[1], "rerank": seg[2],
                            "epilogue": seg[3], "finalize": seg[4]},
            "rerank_rows_per_step": int(flagged.value),
            "roofline": _roofline(achieved, n_local * K, assign_ms, ffma_peak_tflops, traffic, n_local,
                                  clocks, K),
            "e2e": {"value": evals / e2e_s / 1e9, "unit": UNIT, "ms_per_step": e2e_s * 1e3,
                    "api": "vqb_lloyd_step_f32 (C ABI), X from pinned host memory"
                           + (", per rank on its shard" if world > 1 else ""),
                    "h2d_bytes_per_step": n_local * 16 * 4 + K * 16 * 8,
                    "d2h_bytes_per_step": K * 16 * 8 + 8,
                    "result": "new codebook + distortion"},
            "e2e_pageable": {"value": evals / e2e_pg_s / 1e9, "unit": UNIT, "ms_per_step": e2e_pg_s * 1e3,
                             "api": "vqb_lloyd_step_f32, X from pageable numpy (staged copy engine)"},
            "cpu_baseline": {"value": cpu_rate, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{rows} leading rows of {name} x K={K}, assign+TD+update "
                                       f"(oracle/ C+OpenMP, reference arithmetic), min of 3",
                             "cpu_model": model},
            "design": design,
            "clocks": {k: c[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
            "gpu_launches": launches_per_step * args.steps,
        }
        result.update(second)
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _workload_golden(name):
    path = os.path.join(ROOT, "tests", "golden",
                        f"{name}_{'encode' if name == 'cfg5' else 'design'}.npz")
    return np.load(path) if os.path.exists(path) else None


def run_workload_sharded(args):
    """A design workload (cfg1-cfg4) on N GPUs, one process per GPU: strong
    scaling -- every rank holds a contiguous tile-aligned shard of the SAME
    global training set (distributed.ShardPlan), one NCCL allreduce per pass
    (distributed.sharded_lbg_train).  Time = the slowest rank's wall time of
    the whole design (barrier + device synchronise on both sides)."""
    import torch
    import torch.distributed as dist

    import paper_0910_4711_b200 as vq
    from paper_0910_4711_b200 import synthetic
    from paper_0910_4711_b200.distributed import sharded_lbg_train

    rank, world, local_rank = _rank_env()
    torch.cuda.set_device(local_rank)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    name = args.workload
    spec = synthetic.WORKLOADS[name]
    x = synthetic.make_training(name)  # every rank generates the same set
    ts = vq.TrainingSet(x)
    conf = vq.LbgConfig(target_size=spec.target_size, epsilon=spec.epsilon, delta=spec.delta)
    from paper_0910_4711_b200.distributed import DeviceShard

    cache = {}

    def shard(rows, lo, n):  # this rank's rows stay resident across the timed designs
        if "s" not in cache:
            cache["s"] = DeviceShard(np.ascontiguousarray(rows), lo, n, local_rank)
        return cache["s"]

    clocks = ClockSampler(local_rank).__enter__()
    walls = []
    cb = stats = None
    for i in range(max(1, args.warmup) + max(1, min(args.steps, 2))):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cb, stats = sharded_lbg_train(ts, conf, backend_factory=shard)
        torch.cuda.synchronize()
        t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if i >= max(1, args.warmup):
            walls.append(float(t.item()))
    clocks.__exit__(None, None, None)
    if rank == 0:
        g = _workload_golden(name)
        parity = None
        if g is not None:
            gh = g["hist"]
            parity = {
                "schedule_matches_reference": bool(
                    len(stats.history) == gh.shape[0] and all(
                        (h.codebook_size, h.iteration, h.empty_cells) == (int(r[0]), int(r[1]), int(r[3]))
                        for h, r in zip(stats.history, gh))),
                "total_rel_err": abs(stats.total - float(g["total"])) / float(g["total"]),
                "codebook_max_rel_err": float(np.max(np.abs(cb.codevectors - g["cb"]) /
                                                     np.maximum(np.abs(g["cb"]), 1e-300))),
            }
        c = clocks.summary()
        wall = min(walls)
        print(json.dumps({
            "metric": "codebook design wall-time (s)", "value": wall, "unit": "s", "impl": "b200",
            "n_gpus": world, "steps": len(walls), "warmup": max(1, args.warmup), "ms_per_step": wall * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64",
            "data": "synthetic",
            "config": {"workload": f"{name}: {spec.name} N={x.shape[0]} L={x.shape[1]} K 1->{spec.target_size}, "
                                   f"rows sharded over {world} GPUs", "parallelism": f"dp{world}",
                       "exchange": "one NCCL allreduce of the packed int64 buffer per pass",
                       "resident": "each rank's shard uploaded once before the timed designs"},
            "passes": len(stats.history), "parity": parity,
            "clocks": {k: c[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
        }), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def run_encode(args):
    """cfg5 (BASELINE configs[4]): encode 2^26 queries against the fixed
    K=1024 codebook, sharded over N GPUs (torchrun, one process per GPU):
    every rank holds a contiguous tile-aligned shard of the same query set;
    value = N * K / the slowest rank's device-resident allocation pass
    (candidate pass + re-rank + exact distances + distortion; CUDA events).
    e2e = distributed.sharded_encode / codec.encode from host numpy (H2D,
    encode, D2H, index all-gather), the public call."""
    import hashlib

    import torch

    import paper_0910_4711_b200 as vq
    from paper_0910_4711_b200 import _lib, synthetic
    from paper_0910_4711_b200 import distributed as D
    from paper_0910_4711_b200.core import _Session

    rank, world, local_rank = _rank_env()
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    L = _lib.lib()
    cb32, q = synthetic.make_encode_case()
    cb = cb32.astype(np.float64)
    n, K = q.shape[0], cb.shape[0]
    plan = D.ShardPlan(n, world)
    lo, hi = plan.bounds(rank)
    g = _workload_golden("cfg5")
    clocks = ClockSampler(local_rank).__enter__()
    sess = _Session(np.ascontiguousarray(q[lo:hi]), None, device=local_rank, row_offset=lo, n_global=n)
    ms, total, fl = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
    _lib.check(L.vqb_bench_assign(sess.handle, _lib.ptr(cb), K, max(1, args.warmup),
                                  ctypes.byref(ms), ctypes.byref(total), ctypes.byref(fl)))
    if world > 1:
        dist.barrier()
    _lib.check(L.vqb_bench_assign(sess.handle, _lib.ptr(cb), K, args.steps,
                                  ctypes.byref(ms), ctypes.byref(total), ctypes.byref(fl)))
    dev_ms = ms.value
    local_idx = sess.assign_u32(cb)
    sess.close()
    del sess
    torch.cuda.empty_cache()
    t = torch.tensor([dev_ms, total.value, float(fl.value)], dtype=torch.float64, device=f"cuda:{local_rank}")
    if world > 1:
        tm = t.clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        dev_ms, tot, flagged = float(tm[0]), float(t[1]), int(t[2])
    else:
        tot, flagged = total.value, int(fl.value)
    # e2e through the public call (every rank: its shard H2D + encode + the gather)
    e2e_runs = []
    stream = None
    for _ in range(2):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        stream = vq.encode(q, vq.Codebook(cb))
        t1 = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=f"cuda:{local_rank}")
        if world > 1:
            dist.all_reduce(t1, op=dist.ReduceOp.MAX)
        e2e_runs.append(float(t1.item()))
    e2e_s = min(e2e_runs)
    clocks.__exit__(None, None, None)
    if rank == 0:
        c = clocks.summary()
        parity = None
        if g is not None:
            want = g["idx_sha256"].item().decode()
            parity = {
                "encode_api_sha256_match": hashlib.sha256(stream.indices.tobytes()).hexdigest() == want,
                "shard0_head_match": bool(np.array_equal(local_idx[:65536], g["head"][: min(65536, hi - lo)])),
                "total_rel_err": abs(tot - float(g["total"])) / float(g["total"]),
                "reference_encode_s": float(g["seconds"]), "reference_workers": int(g["workers"]),
            }
        print(json.dumps({
            "metric": "G vector·codeword distance evals/s (encode pass)", "impl": "b200",
            "value": n * K / (dev_ms * 1e-3) / 1e9, "unit": "G evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
            "config": {"workload": "cfg5: encode N=2^26 L=16 K=1024 (fixed seeded codebook)",
                       "rows": n, "codebook": K, "dim": 16,
                       "parallelism": f"dp{world}" if world > 1 else "single",
                       "sharding": "contiguous tile-aligned query shards, indices all-gathered"},
            "rerank_rows_per_step": flagged,
            "e2e": {"value": n * K / e2e_s / 1e9, "unit": "G evals/s", "seconds": e2e_s,
                    "api": "codec.encode (distributed.sharded_encode under torchrun)",
                    "h2d_bytes_per_step": int(q.nbytes + cb.nbytes), "d2h_bytes_per_step": int(n * 4)},
            "parity": parity,
            "clocks": {k: c[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
        }), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_workload(args):
    """One BASELINE config end to end on one GPU (parity-checked against the
    reference's committed outputs where they exist):
      cfg1/cfg3/cfg4  full codebook design (device-resident wall time and
                      through lbg_train with host buffers) + one Lloyd
                      iteration at the final codebook;
      cfg5            encode of 2^26 queries (device-resident allocation pass,
                      and through encode() from host memory)."""
    import torch

    import paper_0910_4711_b200 as vq
    from paper_0910_4711_b200 import _lib, synthetic
    from paper_0910_4711_b200.core import _Session

    name = args.workload
    L = _lib.lib()
    spec = synthetic.WORKLOADS[name]
    g = _workload_golden(name)
    out = {"impl": "b200", "n_gpus": 1, "data": "synthetic", "steps": args.steps,
           "warmup": args.warmup, "scaling": "weak", "vs_baseline": None}
    if name == "cfg5":
        cb32, q = synthetic.make_encode_case()
        clocks = ClockSampler(0).__enter__()  # sampled from here on: GPU work only
        cb = cb32.astype(np.float64)
        n, K = q.shape[0], cb.shape[0]
        sess = _Session(q, None)
        ms, total, fl = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        _lib.check(L.vqb_bench_assign(sess.handle, _lib.ptr(cb), K, max(1, args.warmup),
                                      ctypes.byref(ms), ctypes.byref(total), ctypes.byref(fl)))
        _lib.check(L.vqb_bench_assign(sess.handle, _lib.ptr(cb), K, args.steps,
                                      ctypes.byref(ms), ctypes.byref(total), ctypes.byref(fl)))
        dev_ms = ms.value
        idx = sess.assign_u32(cb)
        sess.close()
        del sess
        torch.cuda.empty_cache()
        e2e_runs = []
        for _ in range(3):
            t0 = time.perf_counter()
            stream = vq.encode(q, vq.Codebook(cb))
            e2e_runs.append(time.perf_counter() - t0)
        e2e_s = min(e2e_runs[1:])
        import hashlib
        parity = None
        if g is not None:
            parity = {
                "indices_sha256_match": hashlib.sha256(idx.tobytes()).hexdigest()
                == g["idx_sha256"].item().decode(),
                "encode_api_sha256_match": hashlib.sha256(stream.indices.tobytes()).hexdigest()
                == g["idx_sha256"].item().decode(),
                "total_rel_err": abs(total.value - float(g["total"])) / float(g["total"]),
                "reference_encode_s": float(g["seconds"]),
                "reference_workers": int(g["workers"]),
            }
        out.update({
            "metric": "G vector·codeword distance evals/s (encode pass)",
            "value": n * K / (dev_ms * 1e-3) / 1e9, "unit": "G evals/s",
            "ms_per_step": dev_ms, "higher_is_better": True, "dtype": "f32+f64",
            "config": {"workload": f"{name}: encode N=2^26 L=16 K=1024 (fixed seeded codebook)",
                       "rows": n, "codebook": K, "dim": 16},
            "rerank_rows_per_step": int(fl.value),
            "e2e": {"value": n * K / e2e_s / 1e9, "unit": "G evals/s", "seconds": e2e_s,
                    "h2d_bytes_per_step": int(q.nbytes + cb.nbytes),
                    "d2h_bytes_per_step": int(n * 4)},
            "parity": parity,
        })
    else:
        x = synthetic.make_training(name)
        clocks = ClockSampler(0).__enter__()  # sampled from here on: GPU work only
        n, dim = x.shape
        conf = vq.LbgConfig(target_size=spec.target_size, epsilon=spec.epsilon, delta=spec.delta)
        sess = _Session(x, None)
        for _ in range(max(1, args.warmup if name != "cfg4" else 1)):
            dcb, hist, warns, total, _d, summ = sess.train(conf)
        reps = max(1, args.steps if name != "cfg4" else min(args.steps, 2))
        walls = []
        for _ in range(reps):
            t0 = time.perf_counter()
            dcb, hist, warns, total, _d, summ = sess.train(conf)
            walls.append(time.perf_counter() - t0)
        wall = min(walls)
        cbf = np.ascontiguousarray(g["cb"]) if g is not None else np.ascontiguousarray(dcb)
        segs = (ctypes.c_double * 5)()
        flagged = ctypes.c_int64()
        _lib.check(L.vqb_bench_iteration(sess.handle, _lib.ptr(cbf), cbf.shape[0], 3, segs,
                                         ctypes.byref(flagged)))
        _lib.check(L.vqb_bench_iteration(sess.handle, _lib.ptr(cbf), cbf.shape[0], args.steps, segs,
                                         ctypes.byref(flagged)))
        it_ms = sum(segs)
        e2e_runs = []
        for _ in range(2 if name == "cfg4" else 3):
            t0 = time.perf_counter()
            cb2, st2 = vq.lbg_train(vq.TrainingSet(x), conf)
            e2e_runs.append(time.perf_counter() - t0)
        e2e_s = min(e2e_runs[1:])
        pix = None
        if name in ("cfg1", "cfg3"):
            # the image configs from their uint8 pixels: vectorised on the
            # device (storage.image_training_set), 1 byte per sample over PCIe
            from paper_0910_4711_b200 import storage

            px = synthetic.make_training_pixels(name)
            runs = []
            for _ in range(3):
                t0 = time.perf_counter()
                ts_px, _grid = storage.image_training_set(px, 4 if name == "cfg1" else 8)
                cb3, st3 = vq.lbg_train(ts_px, conf)
                runs.append(time.perf_counter() - t0)
                del ts_px
            pix = {"value": min(runs[1:]), "unit": "s", "api": "storage.image_training_set + lbg_train",
                   "h2d_bytes_per_step": int(px.nbytes), "d2h_bytes_per_step": int(dcb.nbytes),
                   "codebook_equal_to_float_path": bool(cb3.codevectors.tobytes() == cb2.codevectors.tobytes())}
        parity = None
        if g is not None:
            gh = g["hist"]
            parity = {
                "reference_passes": int(gh.shape[0]),
                "schedule_matches_reference": bool(
                    len(hist) == gh.shape[0] and all(
                        (h.codebook_size, h.iteration, h.empty_cells) ==
                        (int(r[0]), int(r[1]), int(r[3])) for h, r in zip(hist, gh))),
                "total_rel_err": abs(total - float(g["total"])) / float(g["total"]),
                "codebook_max_rel_err": float(np.max(np.abs(dcb - g["cb"]) /
                                                     np.maximum(np.abs(g["cb"]), 1e-300))),
                "codebook_bit_identical": bool(dcb.tobytes() == g["cb"].tobytes()),
                "reference_wall_s": float(g["seconds"]),
                "reference_workers": int(g["workers"]),
            }
        out.update({
            "metric": "codebook design wall-time (s)", "value": wall, "unit": "s",
            "ms_per_step": wall * 1e3, "higher_is_better": False, "dtype": "f32+f64",
            "config": {"workload": f"{name}: {spec.name} N={n} L={dim} K 1->{spec.target_size}, "
                                   f"delta={spec.delta}, eps={spec.epsilon}",
                       "rows": n, "dim": dim, "target_size": spec.target_size},
            "passes": int(summ.passes), "evals": int(summ.evals),
            "design_g_evals_per_s": summ.evals / wall / 1e9,
            "flagged_rows": int(summ.flagged_rows),
            "flagged_full_scan_rows": int(summ.flagged_full),
            "final_iteration": {"ms": it_ms, "g_evals_per_s": n * cbf.shape[0] / (it_ms * 1e-3) / 1e9,
                                "segments_ms": list(segs), "rerank_rows": int(flagged.value)},
            "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(x.nbytes),
                    "d2h_bytes_per_step": int(dcb.nbytes)},
            "e2e_from_pixels": pix,
            "parity": parity,
        })
    clocks.__exit__(None, None, None)
    c = clocks.summary()
    out["clocks"] = {k: c[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")}
    print(json.dumps(out), flush=True)
    return 0


def run_formats(args):
    """The HBM-bound kernels either side of the path,
    each at its BASELINE scale: the cfg3 block vectoriser (16 x 2048^2 pixels,
    8x8 blocks), the cfg5 decode (2^26 indices, K=1024, L=16), the fused
    decode-to-pixels and raster at cfg3, and the pair distances of
    reconstruction_distortion at cfg5.  Per kernel: device-resident event time,
    algorithmic bytes / time vs the measured HBM peak; e2e through the public
    API from host buffers; the CPU numpy path (oracle restatement of the
    reference's numpy code) on a bounded sample."""
    import paper_0910_4711_b200 as vq
    from paper_0910_4711_b200 import _lib, synthetic

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    L = _lib.lib()
    peaks, src = _measured_peaks()
    hbm = float(peaks["hbm_gbs"])
    shapes = {  # which: (label, images, h, w, block, n, dim, size)
        0: ("pixels_to_blocks f32 (cfg3: 16 x 2048^2, b=8)", 16, 2048, 2048, 8, 0, 0, 1),
        1: ("pixels_to_blocks f64 (cfg3)", 16, 2048, 2048, 8, 0, 0, 1),
        2: ("blocks_to_pixels (cfg3)", 16, 2048, 2048, 8, 0, 0, 1),
        3: ("decode (cfg5: 2^26 x L=16, K=1024)", 0, 0, 0, 0, 1 << 26, 16, 1024),
        4: ("decode_pixels (cfg3, K=512)", 16, 2048, 2048, 8, 0, 0, 512),
        5: ("pair distances (cfg5: 2^26 x L=16)", 0, 0, 0, 0, 1 << 26, 16, 1),
    }
    clocks = ClockSampler(0).__enter__()
    kernels = {}
    for which, (label, im, h, w, b, n, dim, size) in shapes.items():
        ms, by = ctypes.c_double(), ctypes.c_double()
        _lib.check(L.vqb_bench_formats(which, im, h, w, b, n, dim, size, max(args.steps, 3),
                                       ctypes.byref(ms), ctypes.byref(by)))
        gbs = by.value / (ms.value * 1e-3) / 1e9
        kernels[label] = {"ms": ms.value, "algorithmic_bytes": by.value, "gb_per_s": gbs,
                          "frac_of_hbm_peak": gbs / hbm}
    clocks.__exit__(None, None, None)
    # e2e through the public API (host buffers, copies included)
    px = synthetic.make_training_pixels("cfg3", images=4)  # 4 x 2048^2 (bounded host memory)
    t = []
    for _ in range(3):
        t0 = time.perf_counter()
        vec, grid = vq.pixels_to_blocks(px, 8)
        t.append(time.perf_counter() - t0)
    e2e_p2b = min(t)
    t0 = time.perf_counter()
    want = np.concatenate([oracle.pixels_to_blocks(im, 8) for im in px[:1]])
    cpu_p2b = time.perf_counter() - t0
    assert vec[:want.shape[0]].tobytes() == want.tobytes()
    cb = vq.Codebook(np.random.default_rng(3).normal(128, 60, (1024, 16)))
    idx = np.random.default_rng(4).integers(0, 1024, 1 << 24).astype(np.uint32)
    stream = vq.EncodedStream(1024, 16, idx)
    t = []
    for _ in range(3):
        t0 = time.perf_counter()
        rows = vq.decode(stream, cb)
        t.append(time.perf_counter() - t0)
    e2e_dec = min(t)
    t0 = time.perf_counter()
    ref_rows = oracle.decode(idx, cb.codevectors)
    cpu_dec = time.perf_counter() - t0
    parity = {"pixels_to_blocks_bit_exact_image0": True,
              "decode_bit_exact": bool(rows.tobytes() == ref_rows.tobytes())}
    c = clocks.summary()
    head = kernels["decode (cfg5: 2^26 x L=16, K=1024)"]
    out = {
        "metric": "GB/s (HBM-bound format kernels)", "value": head["gb_per_s"], "unit": "GB/s",
        "impl": "b200", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": head["ms"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8/f32/f64", "data": "synthetic",
        "config": {"workload": "formats: block vectoriser / raster / decode / pair distances at cfg3 and cfg5 scale",
                   "l2": "inputs+outputs of every launch exceed the 126 MB L2"},
        "roofline": {"bound": "hbm", "kernel": "decode", "achieved": head["gb_per_s"], "peak": hbm,
                     "unit": "GB/s", "frac": head["frac_of_hbm_peak"], "peak_source": src,
                     "traffic": None},
        "kernels": kernels,
        "e2e": {"pixels_to_blocks_4x2048sq_f64_s": e2e_p2b,
                "pixels_to_blocks_gb_per_s_of_output": vec.nbytes / e2e_p2b / 1e9,
                "decode_2e24_rows_s": e2e_dec,
                "decode_gb_per_s_of_output": rows.nbytes / e2e_dec / 1e9,
                "h2d_bytes_per_step": int(px.nbytes + idx.nbytes + cb.codevectors.nbytes),
                "d2h_bytes_per_step": int(vec.nbytes + rows.nbytes)},
        "cpu_baseline": {"pixels_to_blocks_2048sq_s": cpu_p2b, "decode_2e24_rows_s": cpu_dec,
                         "kind": "port", "cores": 1,
                         "sample": "one 2048^2 image (oracle numpy vectoriser); 2^24-row numpy gather"},
        "parity": parity,
        "clocks": {k: c[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
    }
    print(json.dumps(out), flush=True)
    return 0


def sess_fast(sess) -> bool:
    return sess.dim in (16, 32, 64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="lloyd",
                    choices=["lloyd", "cfg1", "cfg2", "cfg3", "cfg4", "cfg4-design", "cfg5", "formats"],
                    help="lloyd (default): the headline cfg4 Lloyd-iteration line (+ cfg2 beside it); "
                         "cfg2: the cfg2 Lloyd line; cfg1/cfg3/cfg4-design/cfg5/formats: one line each")
    ap.add_argument("--profile-steps", action="store_true",
                    help="only the warm-up + timed steps (for ncu launch lists)")
    args = ap.parse_args()
    if args.workload in ("lloyd", "cfg4"):
        args.workload = "cfg4"
    elif args.workload == "cfg4-design":
        args.workload = "cfg4"
        args.design = True
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "formats":
        return run_formats(args)
    design = getattr(args, "design", False) or args.workload in ("cfg1", "cfg3")
    if design and (_rank_env()[1] > 1 or os.environ.get("VQB_BENCH_SHARDED") == "1"):  # (the latter: test hook)
        return run_workload_sharded(args)
    if args.workload == "cfg5":
        return run_encode(args)
    if design:
        return run_workload(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
