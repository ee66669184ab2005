#!/usr/bin/env python
"""Benchmark: RASTER contraction + agglomeration on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 4] [--order gen|shuffled] [--quick]

One step = cluster_sequential over the whole workload: K1 contraction, K2
compaction, K3 connected components + mu filter + canonical ids (results
device-resident). Headline workload: BASELINE config 4 (500M float64 points,
8 GB, 1,000,000 Gaussian clusters x 500, sigma 5e-4, p=3, tau=4, mu=4) in
generation order; inputs (8 GB) exceed the 126 MB L2, so no flush is needed
between steps.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse

import numpy as np
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "points/sec clustered at 1 B200 (contraction+agglomeration); % of HBM roofline"
BYTES_PER_POINT = 16  # algorithmic: read (x, y) float64 once
WORKLOADS = {
    1: "config1: 1M pts, 1,000 Gaussian clusters x 1,000 (sigma 0.005), p=2 tau=5 mu=4",
    2: "config2: 10M pts, 10,000 clusters x 900 (sigma 0.005) + 1M uniform noise, p=2 tau=5 mu=4",
    3: "config3: 100M pts, 100,000 clusters x 1,000 (sigma 5e-4), p=3 tau=5 mu=4",
    4: "config4: 500M pts (8 GB), 1,000,000 Gaussian clusters x 500 (sigma 5e-4), p=3 tau=4 mu=4",
    5: "config5: 200M pts, 100M blob (sigma 1e-4) + 1,000 walks x 20,000 steps x 3 + 40M noise, p=3 tau=3 mu=4",
}


def measured_peak_gbs() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        v = float(json.loads(p.read_text())["hbm_gbs"])
        return v, "measured (MEASURED_PEAKS.json hbm_gbs, copy test)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML every ~5 ms while
    the timed region runs (the recipe's nvidia-smi clocks line, at a rate
    that also covers short regions; a 2 ms period measurably slowed the
    launch thread through the GIL)."""

    REASONS = {
        "hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
        "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
        "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
        "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
        "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown",
    }

    def __init__(self, index: int, period_s: float = 0.005):
        self.index = index
        self.period = period_s
        self.sm: list[float] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception as e:  # NVML missing: report no samples
            self.err = str(e)
        return self

    def _run(self):
        nv = self.nv
        masks = {k: getattr(nv, v) for k, v in self.REASONS.items() if hasattr(nv, v)}
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, m in masks.items():
                    if r & m:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "NVML, 5 ms period, timed region only"}


def k1_traffic(n: int):
    """dram bytes per K1 launch from the committed ncu --set full capture
    (profiles/r02/k1_traffic.json), scaled to this workload; None if absent."""
    try:
        d = json.loads((ROOT / "profiles" / "r02" / "k1_traffic.json").read_text())
        return d["traffic_bytes_per_launch"] * n / (d["algorithmic_bytes_per_launch"] / BYTES_PER_POINT)
    except Exception:
        return None


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def host_cpu() -> dict:
    """nproc and the lscpu model name of this host."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count() or 1, "model": model}


def reference_arm(args) -> None:
    """The reference's own CPU implementation (oracle/_ref = the reference
    compiled from its headers, raster::cluster_parallel with every host
    thread) on the SAME workload as our arm (the full config by default).
    When K full-size runs would not fit --ref-budget-s, fewer are timed and
    the line says so (steps, steps_requested)."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    from oracle import pyoracle as O
    from paper_1907_03620_b200 import datagen as D

    if O.ref() is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libraster_ref.so not built"}))
        return
    cores = os.cpu_count() or 1
    workers = args.ref_workers if args.ref_workers is not None else cores
    s = D.spec(args.config)
    per = s.points_per_cluster
    full = D.count(s)
    if args.ref_sample and args.ref_sample < full:
        # bounded sample = the first clusters of the workload (generation order)
        s.n_clusters = max(1, args.ref_sample // max(per, 1)) if per else s.n_clusters
    pts = D.generate(s, shuffle_seed=(11 if args.order == "shuffled" else None))
    n = pts.shape[0]
    gp = D.params(args.config)
    t_start = time.perf_counter()
    warm = []
    for _ in range(max(1, args.warmup)):
        warm.append(O.ref_time(pts.ctypes.data, n, gp, workers)[0])
        if time.perf_counter() - t_start > args.ref_budget_s / 4:
            break
    per_run = min(warm)
    steps = max(1, min(args.steps, int(args.ref_budget_s // max(per_run, 1e-9))))
    times = [O.ref_time(pts.ctypes.data, n, gp, workers)[0] for _ in range(steps)]
    med = statistics.median(times)
    value = n / med
    what = (f"all {n:,} points" if n == full else f"first {n:,} points ({s.n_clusters:,} clusters)")
    sample = (f"{what} of {WORKLOADS[args.config].split(':')[0]} ({full:,} points), {args.order} order; "
              f"raster::cluster_{'parallel' if workers else 'sequential'} count mode; median of "
              f"{steps} timed runs after {len(warm)} warm-up")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s",
        "n_gpus": world, "steps": steps, "steps_requested": args.steps, "warmup": len(warm),
        "ms_per_step": med * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "order": args.order, "points": n,
                   "same_config": n == full,
                   "parallelism": f"cpu x{max(workers, 1)} threads"},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": max(workers, 1),
                         "kind": "reference", "sample": sample, "host": host_cpu(),
                         "runs_s": times},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def cpu_baseline_sequential(pts_host, gp, n_count: int, n_retain: int) -> dict:
    """The reference's cluster_sequential on 1 core: count mode over
    n_count points (the whole workload by default, one run) and
    Mode::retain_points (the point-retaining variant) over the first
    n_retain points."""
    from oracle import pyoracle as O

    if O.ref() is None:
        t0 = time.perf_counter()
        O.port_cluster(pts_host[:n_count], gp)
        t = time.perf_counter() - t0
        return {"value": n_count / t, "unit": "points/s", "cores": 1, "kind": "port",
                "sample": f"first {n_count:,} points, oracle port, 1 thread", "host": host_cpu()}
    t, tp, tc, _ = O.ref_time(pts_host.ctypes.data, n_count, gp, 0)
    out = {"value": n_count / t, "unit": "points/s", "cores": 1, "kind": "reference",
           "sample": (f"{'all' if n_count == len(pts_host) else 'first'} {n_count:,} points of the "
                      "workload (generation order), raster::cluster_sequential count mode, "
                      "1 thread, 1 run"),
           "same_config": n_count == len(pts_host),
           "phases_s": {"projection": tp, "clustering": tc}, "host": host_cpu()}
    if n_retain:
        tr, _, _, _ = O.ref_time_mode(pts_host.ctypes.data, n_retain, gp, 0, True)
        out["retain_points"] = {
            "value": n_retain / tr, "unit": "points/s", "cores": 1,
            "sample": f"first {n_retain:,} points, raster::cluster_sequential Mode::retain_points, "
                      "1 thread, 1 run (the reference's point-retaining variant)"}
    return out


def stream_leg(gp, pts) -> dict:
    """The chunked PointSource path (rg_stream_*, io.hpp:226-241): a
    memory-backed source whose read() copies the next chunk into the pinned
    staging buffer, while the previous chunk's H2D copy and K1 run. Host
    wall clock from the first read to the last chunk's contraction (the
    source's copies are part of the job, as a file read would be)."""
    from paper_1907_03620_b200.raster import TileAccumulator

    chunk = 1 << 22
    acc = TileAccumulator(gp)
    pos = [0]

    def read(out):
        k = min(len(out), len(pts) - pos[0])
        np.copyto(out[:k], pts[pos[0]:pos[0] + k])
        pos[0] += k
        return k

    acc.ingest_source(read, chunk)  # warm-up (buffers, table)
    del acc
    pos[0] = 0
    acc2 = TileAccumulator(gp)
    acc2.ingest_source(lambda out: 0, chunk)
    t0 = time.perf_counter()
    n = acc2.ingest_source(read, chunk)
    t = time.perf_counter() - t0
    assert acc2.total_ingested() + acc2.skipped() == len(pts)
    return {"points_per_s": n / t, "seconds": t, "chunk_points": chunk,
            "source": "memory-backed PointSource: read() = numpy copy of the next chunk into the "
                      "pinned buffer (single host thread), overlapped with the previous chunk's "
                      "H2D + K1"}


def per_config_sweep(args, pl4, stream, dev4) -> dict:
    """Every BASELINE config (1-5), in generation order and in a seeded random
    order (device permutation): device time per rg_cluster call with the
    points resident, points/s and the fraction of the 16 B/pt roofline."""
    import torch

    from paper_1907_03620_b200 import datagen as D
    from paper_1907_03620_b200.raster import Pipeline

    peak, _ = measured_peak_gbs()
    out = {}
    for cfg in (1, 2, 3, 4, 5):
        if cfg == 4 and dev4 is not None:
            dev, pl = dev4, pl4
        else:
            dev = torch.from_numpy(D.generate(D.spec(cfg))).to(stream.device)
            pl = Pipeline(D.params(cfg), device=stream.device.index)
            pl.set_stream(stream.cuda_stream)
        n = dev.shape[0]
        g = torch.Generator(device=dev.device)
        g.manual_seed(11)
        for order in ("gen", "shuffled"):
            x = dev if order == "gen" else dev[torch.randperm(n, device=dev.device, generator=g)]
            for _ in range(max(3, args.warmup)):
                pl.run(x)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            k1 = []
            e0.record(stream)
            for _ in range(args.steps):
                k1.append(pl.run(x).ms_contract)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            k1_ms = statistics.mean(k1)
            out[f"config{cfg}_{order}"] = {
                "points": n, "ms_per_step": ms, "points_per_s": n / (ms / 1e3),
                "roofline_frac": (BYTES_PER_POINT * n / (ms / 1e3) / 1e9) / peak,
                "contract_ms": k1_ms,
                "contract_frac": (BYTES_PER_POINT * n / (k1_ms / 1e3) / 1e9) / peak}
            del x
        del dev
    return out


def ours(args) -> None:
    import numpy as np
    import torch

    from paper_1907_03620_b200 import datagen as D
    from paper_1907_03620_b200.raster import Pipeline

    rank, local, world = dist_env()
    # RG_BENCH_BACKEND=gloo RG_BENCH_SAME_GPU=1: exercise the N>1 code path
    # with several ranks on one GPU (a functional check, never a measurement)
    backend = os.environ.get("RG_BENCH_BACKEND", "nccl")
    if os.environ.get("RG_BENCH_SAME_GPU"):
        local = 0
    torch.cuda.set_device(local)
    red_dev = "cuda" if backend == "nccl" else "cpu"
    dist = None
    if world > 1:
        import torch.distributed as dist_mod

        dist_mod.init_process_group(backend)
        dist = dist_mod
    cfg = args.config
    s = D.spec(cfg)
    if world > 1:  # weak scaling: each rank clusters its own seeded shard
        s.seed = s.seed + 7919 * rank
    n = D.count(s)
    gp = D.params(cfg)

    host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
    t0 = time.perf_counter()
    D.generate_into(s, host.data_ptr())
    if args.order == "shuffled":
        host.numpy()[:] = D.shuffle(host.numpy(), 11)
    t_gen = time.perf_counter() - t0
    dev = host.to(f"cuda:{local}", non_blocking=False)
    stream = torch.cuda.current_stream()
    if world == 1:
        pl = Pipeline(gp, device=local)
        pl.set_stream(stream.cuda_stream)
        result_ctx = pl.ctx
        launches_of = pl.launches
    else:
        # N>1: the union of all ranks' shards is clustered: counts routed to
        # the owner of their column range (NCCL all_to_all), each owner prunes
        # and agglomerates its own columns, border join (distributed.py)
        from paper_1907_03620_b200.distributed import DistributedPipeline

        pl = DistributedPipeline(gp, device=local, stream=stream.cuda_stream)
        result_ctx = pl.engine.owner
        launches_of = pl.engine.launches

    def step_stats(ret):
        """(ms_contract, rg_stats-like facts) of the step just run."""
        if world == 1:
            return ret.ms_contract, ret
        loc, own = pl.engine.local.stats(), result_ctx.stats()
        own.ms_contract, own.peak_accumulator_entries = loc.ms_contract, loc.peak_accumulator_entries
        own.n_significant = ret.n_significant
        own.n_clusters = pl.stats_n_clusters
        return loc.ms_contract, own

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        pl.run(dev)
    barrier()
    launches0 = launches_of()
    ms_contract = []
    st = None
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            mc, st = step_stats(pl.run(dev))
            ms_contract.append(mc)
        e1.record(stream)
        barrier()
    launches = launches_of() - launches0
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = n * world / (ms_step / 1e3)

    # e2e: through the public API from pinned host memory, reading the
    # canonical result (sorted significant tiles + counts + cluster ids) back.
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    S = st.n_significant if world == 1 else int(pl.part[0].numel())  # this rank's columns
    # the result lands in pinned host buffers (as the input comes from one)
    pinned = [torch.empty(max(S, 1), dtype=torch.int64, pin_memory=True) for _ in range(4)]
    tx, ty, cnt, cid = (p.numpy() for p in pinned)
    from paper_1907_03620_b200 import _native as N

    def readback():
        if world == 1:
            result_ctx.check(result_ctx.lib.rg_get_significant(
                result_ctx.h, tx.ctypes.data, ty.ctypes.data, cnt.ctypes.data, cid.ctypes.data, S,
                N.RG_MEM_HOST))
        else:  # this rank's columns of the canonical result (global ids)
            for dst, src in zip(pinned, pl.part):
                dst[: src.numel()].copy_(src, non_blocking=True)
            torch.cuda.current_stream().synchronize()

    # untimed: the first host-path call allocates the staging buffers, the
    # first readback the result buffers
    pl.run(host)
    readback()
    barrier()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(e2e_steps):
        pl.run(host)
        readback()
    f1.record(stream)
    barrier()
    ms_e2e = f0.elapsed_time(f1) / e2e_steps
    if dist:
        t = torch.tensor([ms_e2e], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    e2e_value = n * world / (ms_e2e / 1e3)

    extra = {}
    if not args.quick and world == 1:
        # point-retaining variant: + per-point int32 labels (20 B/pt algorithmic)
        labels = torch.empty(n, dtype=torch.int32, device=dev.device)
        pl.run(dev)
        pl.label_points(dev, labels)
        torch.cuda.synchronize()
        l0 = torch.cuda.Event(enable_timing=True)
        l1 = torch.cuda.Event(enable_timing=True)
        l0.record(stream)
        for _ in range(args.steps):
            pl.run(dev)
            pl.label_points(dev, labels)
        l1.record(stream)
        torch.cuda.synchronize()
        ms_l = l0.elapsed_time(l1) / args.steps
        peak, _ = measured_peak_gbs()
        # 20 B/pt is BASELINE's single-pass figure; the labels need the
        # clusters, so the points are read twice: 36 B/pt compulsory
        extra["labelled"] = {"points_per_s": n / (ms_l / 1e3), "ms_per_step": ms_l,
                             "roofline_frac_20B": (20 * n / (ms_l / 1e3)) / (peak * 1e9),
                             "roofline_frac_two_pass_36B": (36 * n / (ms_l / 1e3)) / (peak * 1e9)}
        del labels
    if not args.quick and world == 1 and args.order == "gen":
        # the same workload in a seeded random order (the reference generator
        # shuffles, datagen.hpp:224-226): no spatial locality for K1's cache;
        # the order probe sends it to the partitioned contraction (K1')
        g = torch.Generator(device=dev.device)
        g.manual_seed(11)
        shuf = dev[torch.randperm(n, device=dev.device, generator=g)]
        for _ in range(args.warmup):
            pl.run(shuf)
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.steps):
            pl.run(shuf)
        s1.record(stream)
        torch.cuda.synchronize()
        ms_s = s0.elapsed_time(s1) / args.steps
        extra["shuffled"] = {"points_per_s": n / (ms_s / 1e3), "ms_per_step": ms_s,
                             "roofline_frac": (BYTES_PER_POINT * n / (ms_s / 1e3))
                             / (measured_peak_gbs()[0] * 1e9),
                             "path": "partitioned contraction: sampled plan + one-pass scatter "
                                     "(k_part_stream), shared-memory aggregation (k_part_agg), "
                                     "pair inserts beside K2/K3",
                             "order": "torch.randperm(seed 11) on the device"}
        del shuf

    if not args.quick and world == 1:
        extra["stream"] = stream_leg(gp, host.numpy())
        extra["per_config"] = per_config_sweep(args, pl, stream, dev if cfg == 4 else None)

    peak, peak_src = measured_peak_gbs()
    k1_ms = statistics.mean(ms_contract)
    achieved = BYTES_PER_POINT * n / (k1_ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, include/raster_datagen.h)",
        "config": {"workload": WORKLOADS[cfg], "order": args.order, "points": n * world,
                   "l2": "inputs 8 GB >> 126 MB L2 each step (no flush needed)" if n >= 100_000_000
                   else "inputs smaller than L2: not flushed",
                   "parallelism": "1 GPU" if world == 1 else
                   f"{world} ranks: own shard each, counts routed to the owner of their "
                   "column range (NCCL all_to_all), K2+K3 per owner on its columns, "
                   "border join of the range edges (small all_gathers)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": k1_traffic(n) if cfg == 4 else None,
                     "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, profiles/r02)",
                     "kernel": "K1 contraction (k_contract), 16 B/point, ms from CUDA events on the launch stream",
                     "peak_source": peak_src,
                     "end_to_end_frac": (BYTES_PER_POINT * n / (ms_step / 1e3) / 1e9) / peak},
        "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": 16 * n,
                "d2h_bytes_per_step": 32 * S},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "phases_ms": {"contract": st.ms_contract, "prune": st.ms_prune,
                      "agglomerate": st.ms_agglomerate},
        "sizes": {"distinct_tiles": st.peak_accumulator_entries, "significant": S,
                  "clusters": st.n_clusters, "table_capacity": st.table_capacity,
                  "grows_total": st.table_grows},
        "gen_seconds": t_gen,
    }
    if extra:
        line["extra"] = extra
    if rank == 0 and world == 1 and not args.no_cpu:
        n_count = min(n, args.cpu_sample) if args.cpu_sample else n
        n_retain = min(n, args.cpu_retain_sample)
        line["cpu_baseline"] = cpu_baseline_sequential(host.numpy(), gp, n_count, n_retain)
    if rank == 0:
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--order", choices=["gen", "shuffled"], default="gen")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="points for the 1-core count-mode baseline (0: the whole workload)")
    ap.add_argument("--cpu-retain-sample", type=int, default=50_000_000,
                    help="points for the 1-core Mode::retain_points baseline (0: skip)")
    ap.add_argument("--ref-sample", type=int, default=0,
                    help="points for the reference arm (0: the whole workload)")
    ap.add_argument("--ref-budget-s", type=float, default=1000.0,
                    help="time budget of the reference arm's timed runs")
    ap.add_argument("--ref-workers", type=int, default=None)
    ap.add_argument("--quick", action="store_true", help="skip the labelled-variant extra")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
