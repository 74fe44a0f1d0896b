#!/usr/bin/env python3
"""Benchmark of the north-star path (BASELINE.json):

  end-to-end DBSCAN Mpoints/s (BVH build + cluster) on configs[1] =
  3D HACC-like clustered halos, 37M points, eps = 0.042, minpts = 2, FDBSCAN,
  one B200 per rank.

One "step" = one full tcg_cluster_device pass (bounds, Morton, radix sort,
Karras topology + refit, fused traversal/union-find, finalize) over the
37M-point cloud, with the points already resident in HBM (the paper's timing
point). `e2e` is the same metric through the reference-facing
C ABI (tc_cluster) with HOST buffers: the H2D copy of the points and the D2H
copy of labels + core flags are inside its timed region.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

N > 1 (torchrun): one global HACC-like cloud of N x 37M points (a slab per
rank) clustered by the Morton-range sharded path (paper_2103_05162_b200/
shard.py: redistribution, eps halo, local passes, cross-shard merge) — weak
scaling; `--replicas` instead runs N independent 37M clouds. Timed as the max
over ranks. (TCB_BENCH_BACKEND=gloo TCB_BENCH_SAME_DEVICE=1 lets a 1-GPU box
smoke-test the N>1 protocol with every rank on cuda:0.)
`--sweep NAME` writes a parameter sweep (the reference's `treeclust bench`
CSV plus device / tc_cluster times and, per row, the reference CPU path on the
same points with a parity verdict) instead of the bench line.
`--impl reference` times the reference's own CPU implementation
(oracle/_ref = /root/reference/proj compiled unmodified) through its public C
ABI on the host cores, on the same 37M-point workload: input from the oracle's
byte-identical generator, loaded with the reference's tc_dataset_load; the
product library is never loaded on that arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

N_POINTS = 37_000_000
EPS = 0.042
MINPTS = 2
ALGO = 0  # TC_ALGO_FDBSCAN
METRIC = "end-to-end DBSCAN Mpoints/s (BVH build+cluster), 3D 37M pts; HBM GB/s"
UNIT = "Mpoints/s"
# algorithmic bytes per point, 3D FDBSCAN minpts=2, one pass.
B_ALG_TOTAL = 183
B_ALG_MAIN = 53  # per traversal pass: leaf coords + node + flag + 2 x parent


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def peaks():
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return None
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx),
                "samples": len(sm), "reasons": sorted(reasons)}


def load_traffic():
    """(dram bytes read + write per launch, limiter evidence) of the main-pass
    kernel from the committed `ncu --set full` summary (profiles/traffic.json)."""
    path = os.path.join(HERE, "profiles", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        lim = dict(t.get("limiter") or {})
        if lim:
            lim["source"] = t.get("source")
        return t.get("k_fd_main_dram_bytes_per_launch"), lim or None
    except Exception:
        return None, None


def reference_input(n):
    """C2's input for the reference arm, made WITHOUT the product library: the
    oracle's byte-identical HACC-like generator (sha256 pinned in
    tests/golden/bench_inputs.json), written in the reference's .bin format and
    loaded through the reference's own tc_dataset_load (REF capi.cpp:84-96)."""
    import shutil
    import tempfile
    from oracle import oracle, ref

    coords = oracle.hacc_like(n)
    tmp = tempfile.mkdtemp(prefix="tcb_ref_")
    try:
        path = os.path.join(tmp, "c2.bin")
        oracle.write_bin(path, coords)
        del coords
        return ref.RefDataset.load(path)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def cpu_reference_times(ds, steps, warmup, threads=0):
    """Wall seconds of the unmodified reference's tc_cluster (REF
    capi.cpp:150-184) on dataset `ds`, plus the last run's stats."""
    times, stats = [], None
    for it in range(warmup + steps):
        dt, stats, _, _ = ds.cluster(EPS, MINPTS, ALGO, threads)
        if it >= warmup:
            times.append(dt)
    return times, stats


def cpu_desc(threads_used):
    from oracle import ref
    return {"cores": threads_used, "host_threads": os.cpu_count() or 1,
            "cpu_model": ref.host_cpu_model()}


def run_reference_arm(args, rank, world):
    """`--impl reference`: the reference's own CPU path (oracle/_ref = the
    unmodified /root/reference/proj compiled from its sources) through its
    public C ABI, on the SAME workload as our arm (C2: 37M HACC-like points,
    eps 0.042, minpts 2, FDBSCAN), threads=0 (all host cores). Rank 0 only."""
    if rank != 0:
        return 0
    steps = max(1, args.steps)
    n = args.points
    t_gen = time.perf_counter()
    ds = reference_input(n)
    t_gen = time.perf_counter() - t_gen
    times, stats = cpu_reference_times(ds, steps, args.warmup)
    ds.close()
    t = sum(times) / len(times)
    value = n / t / 1e6
    desc = cpu_desc(os.cpu_count() or 1)
    sample = (f"the full workload: hacc_like n={n} (oracle generator, .bin via the reference's "
              f"tc_dataset_load, {t_gen:.1f} s), eps={EPS}, minpts={MINPTS}, FDBSCAN, reference "
              f"tc_cluster(threads=0) on {desc['host_threads']} host threads "
              f"({desc['cpu_model']}); per-run s: min {min(times):.2f} max {max(times):.2f}")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 coords / f64 distances", "data": "synthetic",
        "config": {"workload": "C2: 3D HACC-like halos, 37M points, eps=0.042, minpts=2, "
                               "FDBSCAN" if n == N_POINTS else f"C2-shaped, n={n}",
                   "points_per_rank": n, "algorithm": "FDBSCAN", "eps": EPS, "minpts": MINPTS,
                   "parallelism": "host threads (reference parallel_for)"},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": desc["cores"],
                         "cpu_model": desc["cpu_model"], "kind": "reference", "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "stage_s": {k: round(stats[k], 3) for k in ("build_seconds", "preprocess_seconds",
                                                     "main_seconds", "finalize_seconds")},
        "stats": {k: int(stats[k]) for k in ("pair_resolutions", "cluster_count", "core_count",
                                            "noise_count")},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# Parameter sweeps (the reference's `treeclust bench`,
# REF tools/treeclust_cli.cpp:146-198, and the paper's minpts / eps / n
# sweeps): one row per (n, eps, minpts, algorithm) with the
# reference's CSV columns, the device-resident and tc_cluster times, and the
# reference CPU path timed on the same points (this script's reference leg:
# oracle/_ref through dbscan_run, threads = 0) with a parity verdict.
SWEEPS = {
    # name: (generator, n list, eps list, minpts list, algorithms, reference algorithms)
    "hacc-n": ("hacc", [1_000_000, 4_000_000, 16_000_000, 37_000_000], [0.042], [2], [0, 1],
               [0, 1]),
    "hacc-minpts": ("hacc", [4_000_000], [0.042], [2, 5, 10, 50, 100], [0, 1], [0, 1]),
    "hacc-eps": ("hacc", [4_000_000], [0.02, 0.042, 0.084, 0.16], [5], [0, 1], [0, 1]),
    # FDBSCAN on road data resolves ~1e11 pairs at 8M points: the CPU
    # reference is timed for DenseBox only there
    "taxi-minpts": ("taxi", [8_000_000], [0.001], [100, 300, 1000, 3000], [0, 1], [1]),
    "tiny": ("hacc", [20_000, 60_000], [0.042, 0.3], [2, 5], [0, 1], [0, 1]),
}
SWEEP_COLUMNS = ["algorithm", "n", "eps", "minpts", "build_s", "preprocess_s", "main_s",
                 "finalize_s", "total_s", "clusters", "cores", "noise", "dense_fraction",
                 "device_ms", "mpts_per_s", "tc_cluster_ms", "pair_resolutions",
                 "distance_evaluations", "ref_s", "ref_threads", "speedup_vs_ref", "parity"]


def sweep_points(kind, n):
    """The sweep input from the oracle's generators (byte-identical to the
    product's tcg_generate_*): hacc_like keeps C2's density at every n."""
    from oracle import oracle
    return oracle.hacc_like(n) if kind == "hacc" else oracle.taxi_like(n)


def run_sweep(args):
    import csv
    import io

    import numpy as np
    import torch
    import paper_2103_05162_b200 as tb
    from oracle import ref

    kind, n_list, eps_list, minpts_list, algos, ref_algos = SWEEPS[args.sweep]
    names = {0: "fdbscan", 1: "densebox"}
    rows = []
    for n in n_list:
        coords = sweep_points(kind, n)
        ds = tb.Dataset.from_array(coords)
        x = torch.from_numpy(coords).cuda()
        for eps in eps_list:
            for minpts in minpts_list:
                for algo in algos:
                    a = tb.Algorithm(algo)
                    t_abi = float("inf")
                    for _ in range(2):  # the first call also grows the memory pools
                        t0 = time.perf_counter()
                        res = tb.cluster(ds, eps, minpts, a)
                        t_abi = min(t_abi, time.perf_counter() - t0)
                    best = float("inf")
                    for _ in range(3):
                        torch.cuda.synchronize()
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record()
                        tb.cluster_device(x, eps, minpts, a)
                        e1.record()
                        torch.cuda.synchronize()
                        best = min(best, e0.elapsed_time(e1))
                    s = res.stats
                    total = (s["build_seconds"] + s["preprocess_seconds"] + s["main_seconds"]
                             + s["finalize_seconds"])
                    ref_s, parity = None, None
                    if not args.no_ref and algo in ref_algos:
                        t0 = time.perf_counter()
                        want = ref.dbscan(coords, eps, minpts, algo, threads=0)
                        ref_s = time.perf_counter() - t0
                        cm = want["core"] == 1
                        parity = bool(
                            np.array_equal(res.core_flags, want["core"])
                            and np.array_equal(res.labels == -1, want["labels"] == -1)
                            and np.array_equal(res.labels[cm], want["labels"][cm])
                            and all(s[k] == want["stats"][k] for k in (
                                "pair_resolutions", "cluster_count", "core_count",
                                "noise_count")))
                    rows.append([names[algo], n, eps, minpts, s["build_seconds"],
                                 s["preprocess_seconds"], s["main_seconds"], s["finalize_seconds"],
                                 total, s["cluster_count"], s["core_count"], s["noise_count"],
                                 s["dense_point_fraction"], round(best, 3),
                                 round(n / best / 1e3, 2), round(t_abi * 1e3, 3),
                                 s["pair_resolutions"], s["distance_evaluations"],
                                 None if ref_s is None else round(ref_s, 3),
                                 None if ref_s is None else os.cpu_count(),
                                 None if ref_s is None else round(ref_s / t_abi, 1), parity])
                    print(",".join(str(v) for v in rows[-1]), file=sys.stderr, flush=True)
        del ds, x
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(SWEEP_COLUMNS)
    w.writerows(rows)
    if args.sweep_out:
        with open(args.sweep_out, "w") as f:
            f.write(buf.getvalue())
    else:
        sys.stdout.write(buf.getvalue())
    return 0 if all(r[-1] is not False for r in rows) else 1


def run_sharded(args, rank, world, dev, n):
    """N>1: one global HACC-like cloud of world*n points (rank r generates the
    slab x in [r*L, (r+1)*L) with its own seed, same density as C2), clustered
    by the Morton-range sharded path (shard.py): redistribution, eps halo,
    local passes, cross-shard merge. Weak scaling: n points per GPU."""
    import torch
    import torch.distributed as dist
    import paper_2103_05162_b200 as tb
    from paper_2103_05162_b200.shard import DeviceEngine, cluster_sharded

    L = 36.8 * (n / 37e6) ** (1.0 / 3.0)
    c = torch.from_numpy(tb.Dataset.hacc_like(n, box_len=L, seed=11 + rank).coords())
    c[:, 0] += rank * L
    x = c.to(dev)
    gid = (torch.arange(n, dtype=torch.int64) + rank * n).to(dev)
    engine = DeviceEngine(dev)
    for _ in range(args.warmup):
        cluster_sharded(x, gid, EPS, MINPTS, engine)
    torch.cuda.synchronize()
    dist.barrier()
    sampler = ClockSampler(dev.index or 0)
    sampler.start()
    time.sleep(0.3)
    dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    engine.launches = 0
    ev0.record()
    for _ in range(args.steps):
        own_gid, labels, core = cluster_sharded(x, gid, EPS, MINPTS, engine)
    ev1.record()
    torch.cuda.synchronize()
    launches = engine.launches
    dist.barrier()
    clocks = sampler.stop()
    t = torch.tensor([ev0.elapsed_time(ev1)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps
    value = n * world / (ms * 1e-3) / 1e6

    # e2e: the rank's points from pinned host memory -> sharded clustering ->
    # global ids, labels and core flags of its own points back into pinned
    # host buffers (ids and labels as int32: global ids < 2^31), every step.
    host_x = c.pin_memory()
    host_gid = (torch.arange(n, dtype=torch.int64) + rank * n).pin_memory()
    cap = 2 * n
    out_g = torch.empty(cap, dtype=torch.int32).pin_memory()
    out_l = torch.empty(cap, dtype=torch.int32).pin_memory()
    out_c = torch.empty(cap, dtype=torch.uint8).pin_memory()
    e2e_ms, h2d, d2h = [], 0, 0
    for it in range(1 + args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        xd = host_x.to(dev, non_blocking=True)
        gd = host_gid.to(dev, non_blocking=True)
        og, lab, cor = cluster_sharded(xd, gd, EPS, MINPTS, engine)
        k = og.shape[0]
        if k > cap:  # (a rank owning more than twice its input)
            cap = k
            out_g = torch.empty(cap, dtype=torch.int32).pin_memory()
            out_l = torch.empty(cap, dtype=torch.int32).pin_memory()
            out_c = torch.empty(cap, dtype=torch.uint8).pin_memory()
        out_g[:k].copy_(og.to(torch.int32), non_blocking=True)
        out_l[:k].copy_(lab.to(torch.int32), non_blocking=True)
        out_c[:k].copy_(cor, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        if it >= 1:
            e2e_ms.append(e0.elapsed_time(e1))
        h2d = host_x.numel() * 4 + host_gid.numel() * 8
        d2h = k * (4 + 4 + 1)
    # roofline of the local main pass (the last keyed run's stage events on
    # this rank, over its own + ghost points)
    engine.record_stages = True  # one more (untimed) run for the stage events
    cluster_sharded(x, gid, EPS, MINPTS, engine)
    engine.record_stages = False
    stages = engine.last_stages or {}
    main_ms = float(stages.get("main", 0.0))
    n_local = getattr(engine, "last_local_n", n)
    peak, peak_kind = peaks()
    roofline = None
    if main_ms > 0:
        achieved = B_ALG_MAIN * n_local / (main_ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "kernel": "rank 0's local main stage (k_fd_main_fof_q + "
                                              "k_cover_*) of the keyed run",
                    "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "traffic": load_traffic()[0],
                    "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                    "alg_bytes_per_point": B_ALG_MAIN, "main_ms": round(main_ms, 3)}
    te = torch.tensor([sum(e2e_ms) / len(e2e_ms)], device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = n * world / (float(te.item()) * 1e-3) / 1e6
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 coords / f64 distances (exact reference predicate)",
            "data": "synthetic (HACC-like halo slabs, SURVEY.md §8d)",
            "config": {"workload": f"C5-shaped: 3D HACC-like, {n} points per GPU x {world} GPUs, "
                                   "eps=0.042, minpts=2, FDBSCAN, Morton-range sharded",
                       "points_per_rank": n, "parallelism": f"morton-range shards x{world}",
                       "l2": "inputs exceed the 126 MB L2"},
            "clocks": clocks, "gpu_launches": launches,
            "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": round(float(te.item()), 3),
                    "api": "paper_2103_05162_b200.shard.cluster_sharded (host tensors in/out)"},
            # the CPU baseline is a rank-0, N=1 figure (bench contract)
            "cpu_baseline": None, "roofline": roofline,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def relaunch_under_torchrun(ngpus):
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={ngpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--points", type=int, default=N_POINTS, help="points per rank (default: 37M)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph replay leg")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent replicas instead of the Morton-range sharded path")
    ap.add_argument("--sharded", action="store_true",
                    help="run the Morton-range sharded path even at N=1 (its overhead vs the "
                         "direct path)")
    ap.add_argument("--force-exchange", action="store_true",
                    help="sharded path: run the multi-rank protocol (redistribution, halo, merge "
                         "collectives) even on one rank (TCB_SHARD_FORCE_EXCHANGE=1)")
    ap.add_argument("--sweep", choices=sorted(SWEEPS),
                    help="parameter sweep (CSV) with the reference CPU path timed per row")
    ap.add_argument("--sweep-out", help="CSV path for --sweep (default: stdout)")
    ap.add_argument("--no-ref", action="store_true", help="--sweep without the reference column")
    args = ap.parse_args()

    if args.sweep:
        return run_sweep(args)
    if args.force_exchange:
        os.environ["TCB_SHARD_FORCE_EXCHANGE"] = "1"

    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without a launcher: start the N ranks the
        # way the driver does (one process per GPU, torchrun on 127.0.0.1).
        return relaunch_under_torchrun(args.gpus)

    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2103_05162_b200 as tb

    if args.warmup < 3:
        args.warmup = 3
    if os.environ.get("TCB_BENCH_SAME_DEVICE") == "1":
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1 or args.sharded:
        backend = os.environ.get("TCB_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    n = args.points
    if (world > 1 and not args.replicas) or args.sharded:
        return run_sharded(args, rank, world, dev, n)
    # Synthetic HACC-like halos; each rank its own cloud.
    ds = tb.Dataset.hacc_like(n, seed=11 + rank)
    host = torch.from_numpy(ds.coords())
    x = host.to(dev)
    labels = torch.empty(n, dtype=torch.int32, device=dev)
    core = torch.empty(n, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(collect):
        return tb.cluster_device(x, EPS, MINPTS, tb.Algorithm.FDBSCAN, labels, core, stream,
                                 stats=collect)

    for _ in range(args.warmup):
        step(True)
    torch.cuda.synchronize()

    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    stage_sum = {}
    launches = 0
    last_stats = None
    ev0.record(stream)
    for _ in range(args.steps):
        _, _, last_stats = step(True)
        for k, v in tb.last_stage_ms().items():
            stage_sum[k] = stage_sum.get(k, 0.0) + v
        launches += tb.last_launch_count()
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    elapsed_ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    value = n * world / (ms_per_step * 1e-3) / 1e6

    # ---- the same step captured once in a CUDA graph and replayed (FDBSCAN
    # never synchronizes the host, so tcg_cluster_device_async captures) ----
    graph = None
    if not args.no_graph:
        try:
            gl = torch.empty_like(labels)
            gc = torch.empty_like(core)
            gs = torch.empty(1, dtype=torch.int32, device=dev)
            cs = torch.cuda.Stream(dev)
            cs.wait_stream(stream)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cs, capture_error_mode="relaxed"):
                tb.cluster_device_async(x, EPS, MINPTS, tb.Algorithm.FDBSCAN, gl, gc, gs, cs)
            for _ in range(2):
                g.replay()
            torch.cuda.synchronize()
            g0 = torch.cuda.Event(enable_timing=True)
            g1 = torch.cuda.Event(enable_timing=True)
            rs = torch.cuda.current_stream(dev)  # replay() launches on the current stream
            g0.record(rs)
            for _ in range(args.steps):
                g.replay()
            g1.record(rs)
            torch.cuda.synchronize()
            gms = g0.elapsed_time(g1) / args.steps
            cm = core == 1
            graph = {"ms_per_step": round(gms, 3), "value": round(n / (gms * 1e-3) / 1e6, 3),
                     "unit": UNIT, "status": int(gs.item()),
                     "labels_equal": bool(torch.equal(gc, core) and torch.equal(gl[cm], labels[cm])
                                          and torch.equal(gl == -1, labels == -1)),
                     "api": "tcg_cluster_device_async captured once in a CUDA graph, replayed"}
            del g
        except Exception as e:  # reported, never fatal for the bench line
            graph = {"error": str(e)[:200]}

    # ---- e2e through the C ABI with host buffers (H2D + D2H inside) ----
    e2e_times = []
    for it in range(2 + args.steps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        st = tb.cluster_raw(ds, EPS, MINPTS, tb.Algorithm.FDBSCAN)
        dt = time.perf_counter() - t0
        assert st == 0, st
        if it >= 2:
            e2e_times.append(dt)
    e2e_s = sum(e2e_times) / len(e2e_times)
    if world > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = n * world / e2e_s / 1e6

    # ---- CPU baseline: the unmodified reference on the host cores, on the
    # same 37M input (one run, threads=0) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import ref
            rds = ref.RefDataset.from_array(ds.coords())
            times, rstats = cpu_reference_times(rds, 1, 0)
            rds.close()
            tcpu = times[0]
            desc = cpu_desc(os.cpu_count() or 1)
            same = rstats["pair_resolutions"] == (last_stats or {}).get("pair_resolutions")
            cpu = {"value": round(n / tcpu / 1e6, 4), "unit": UNIT, "cores": desc["cores"],
                   "cpu_model": desc["cpu_model"], "kind": "reference",
                   "sample": f"the full workload (n={n}, eps={EPS}, minpts={MINPTS}, FDBSCAN): "
                             f"one reference tc_cluster(threads=0) run, {tcpu:.2f} s; "
                             f"pair_resolutions equal to ours: {same}"}
        except Exception as e:  # the reference .so may be absent on a bare box
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count() or 1,
                   "kind": "reference", "sample": f"unavailable: {e}"}

    steps_n = args.steps
    main_ms = stage_sum.get("main", 0.0) / steps_n
    peak, peak_kind = peaks()
    achieved = (B_ALG_MAIN * n) / (main_ms * 1e-3) / 1e9 if main_ms > 0 else None
    traffic, limiter = load_traffic()
    total_gbs = B_ALG_TOTAL * n / (ms_per_step * 1e-3) / 1e9

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": steps_n, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 coords / f64 distances (exact reference predicate)",
            "data": "synthetic (HACC-like halos, SURVEY.md §8d, seed 11+rank)",
            "config": {"workload": "C2: 3D HACC-like halos, 37M points, eps=0.042, minpts=2, "
                                   "FDBSCAN" if n == N_POINTS else f"C2-shaped, n={n}",
                       "points_per_rank": n, "algorithm": "FDBSCAN", "eps": EPS,
                       "minpts": MINPTS, "parallelism": f"replicas x{world}",
                       "l2": "inputs (444 MB coords + 2.4 GB tree) exceed the 126 MB L2"},
            "stage_ms": {k: round(v / steps_n, 3) for k, v in stage_sum.items()},
            "hbm_gbs_end_to_end": round(total_gbs, 1),
            "roofline": {"bound": "hbm",
                         "kernel": "main stage: k_fd_main_fof_q (fused traversal + warp-batched "
                                   "union-find) + k_cover_* run unions, timed by stage events",
                         "achieved": round(achieved, 1) if achieved else None, "peak": peak,
                         "unit": "GB/s",
                         "frac": round(achieved / peak, 4) if achieved else None,
                         "traffic": traffic,
                         "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                         "alg_bytes_per_point": B_ALG_MAIN,
                         # what actually bounds the traversal (ncu): the L1 data
                         # pipe and the issue slots, not HBM
                         "limiter": limiter},
            "e2e": {"value": round(e2e_value, 3), "unit": UNIT,
                    "h2d_bytes_per_step": n * 3 * 4, "d2h_bytes_per_step": n * 5,
                    "ms_per_step": round(e2e_s * 1e3, 3), "api": "tc_cluster (C ABI)"},
            "graph": graph,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": launches,
            "stats": {k: last_stats[k] for k in ("pair_resolutions", "cluster_count",
                                                  "core_count", "noise_count")}
            if last_stats else None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
