#!/usr/bin/env python3
"""GMACO-P engine benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], the metric's single-GPU config): 32x32
grid road network with signals at every intersection, 1,000 vehicles,
64-ant colonies per vehicle, preemptive signals, congestion-modified
pheromone; one bench step = one colony iteration (every active vehicle's
colony builds 64 complete tours to its destination, then the engine step
B..G advances the world).  Metric: ant-steps/s (one next-hop selection =
one ant-step, counted exactly on the device); vehicle-routes/s alongside.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU code (oracle/_ref, compiled
from /root/reference in place) on the same workload and unit: every active
vehicle's 64 ants walk full tours with the reference's next_node_aco
(routing.cpp:77-115) across all host threads, then the reference's
sequential_step advances its world.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
_RESULT_FD = None


def isolate_stdout() -> None:
    """stdout carries exactly one JSON line: fd 1 is pointed at stderr for
    the whole run (NCCL banners, CUDA / library prints land there) and the
    result line goes to the saved original stdout (emit())."""
    global _RESULT_FD
    sys.stdout.flush()
    _RESULT_FD = os.dup(1)
    os.dup2(2, 1)
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")


def emit(obj) -> None:
    text = json.dumps(obj) + "\n"
    if _RESULT_FD is None:
        sys.stdout.write(text)
        sys.stdout.flush()
    else:
        os.write(_RESULT_FD, text.encode())

import numpy as np  # noqa: E402

GRID = 32
VEHICLES = 1000
ANTS = 64
ITERATIONS = 200
L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=ITERATIONS)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the C4 (1M-node road graph) secondary measurement of the default C2 run")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--config", choices=["c1", "c2", "c3", "c4", "c5"], default="c2",
                    help="BASELINE.json config (c2 = the metric's single-GPU config, the default)")
    ap.add_argument("--skip-extra", action="store_true", help="skip the chained and e2e legs")
    ap.add_argument("--force-comm", action="store_true",
                    help="attach the NCCL exchange even at one rank (exercises the multi-GPU path)")
    ap.add_argument("--algorithm", choices=["colony", "maco-p", "maco", "aco", "dijkstra"], default="colony",
                    help="colony = GMACO-P colonies (the headline); the others run the reference's own "
                         "algorithms (one decision per vehicle at a node per step) on --config c1|c2|c3")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_config(seed: int, max_steps: int, vehicles: int = VEHICLES):
    from paper_2010_14244_b200 import abi
    cfg = abi.default_config(algorithm="colony", controller="preemptive", vehicle_count=vehicles,
                             seed=seed, max_steps=max_steps)
    return abi.colony_production(cfg, ants=ANTS)


def config_block(args, world, vehicles=None):
    from paper_2010_14244_b200 import workloads
    if args.algorithm != "colony":
        R, Cc, sig, V = REF_ALG_SHAPES[args.config]
        return {"workload": f"{args.config.upper()}: {R}x{Cc} grid ({sig} intersections signalized), {V} vehicles, "
                            f"reference algorithm {args.algorithm} (one routing decision per vehicle at a node "
                            f"per step; engine step = sequential_step)",
                "algorithm": args.algorithm, "iterations_timed": args.steps,
                "l2": "flushed (512 MiB write) between timed steps", "parallelism": "1 GPU"}
    if args.config != "c2":
        return {"workload": f"{args.config.upper()}: {workloads.DESCRIPTIONS[args.config]}",
                "vehicles_total": vehicles, "iterations_timed": args.steps,
                "l2": "flushed (512 MiB write) between timed iterations",
                "parallelism": f"one world sharded over {world} GPUs" if world > 1 else "1 GPU"}
    return {
        "workload": "C2: 32x32 grid, signals at every intersection, 1000 vehicles per GPU, 64 ants/colony, "
                    "preemptive signals, one colony iteration per step (GPU arm: congestion-modified roulette and "
                    "best-tour deposit; reference arm: the reference's own next_node_aco tours, which have no "
                    "congestion term, plus its sequential_step)",
        "network": f"grid {GRID}x{GRID}, 200 m edges, 3 lanes, {GRID * GRID} signals",
        "vehicles_per_gpu": VEHICLES,
        "ants_per_colony": ANTS,
        "iterations_timed": args.steps,
        "l2": "flushed (512 MiB write) between timed iterations; working set ~1 MB is L2-resident",
        "parallelism": (f"one world of {VEHICLES * world} vehicles sharded over {world} GPUs (NCCL allgather of "
                        "decisions + int64 allreduce of deposits per step)") if world > 1 else "1 GPU",
    }


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "samples": len(sm), "reasons": sorted(reasons)}


def secondary_c4(peak, peak_src, steps=10, warmup=3):
    """C4 (the north star's 100k-vehicle road-graph config) on the same GPU:
    the HBM-bound ant-queue walker beside the latency-bound C2 headline.
    Same rules as the headline: L2 flushed before each iteration, CUDA events
    (three per iteration here: begin, walk end, step end)."""
    from paper_2010_14244_b200 import workloads
    from paper_2010_14244_b200.engine import Engine
    net, cfg, dist, keep = workloads.c4(seed=1, max_steps=warmup + steps + 1)
    e = Engine(net, cfg, dist)
    e.step(warmup)
    c0 = e.counters()
    walk, stepms = e.bench_steps(steps, L2_FLUSH_BYTES, "both")
    c1 = e.counters()
    e.close()
    del keep
    ant_steps = c1.ant_steps - c0.ant_steps
    alg = c1.walk_bytes - c0.walk_bytes
    walk_s = float(walk.sum()) / 1e3
    achieved = alg / walk_s / 1e9 if walk_s > 0 else 0.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "walk_traffic.json")) as f:
            traffic = json.load(f)["c4"]["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        pass
    return {"workload": "C4: " + workloads.DESCRIPTIONS["c4"], "metric": "ant-steps/sec",
            "value": ant_steps / (float(stepms.sum()) / 1e3), "unit": "ant-steps/s",
            "ms_per_step": float(stepms.mean()), "iterations_timed": steps,
            "vehicle_routes_per_sec": (c1.vehicle_routes - c0.vehicle_routes) / (float(stepms.sum()) / 1e3),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": "k_colony_qt (ant-queue walk over per-target candidate rows; refresh/pro/epi kernels inside the timed walk)",
                         "algorithmic_bytes_per_launch": alg / steps,
                         "avg_launch_us": walk_s / steps * 1e6}}


def secondary_c3(steps=10, warmup=3):
    """C3 (100x100 grid, 10,000 vehicles, 128-ant colonies: the largest
    lattice config of BASELINE.json that one GPU runs whole) on the same GPU,
    same rules as the headline.  No HBM-roofline fraction: the lattice walk's
    state is SMEM/L2-resident, so the byte model does not bound it (its ncu
    limiter is recorded under profiles/)."""
    from paper_2010_14244_b200 import workloads
    from paper_2010_14244_b200.engine import Engine
    net, cfg, dist, keep = workloads.c3(seed=1, max_steps=warmup + steps + 1)
    e = Engine(net, cfg, dist)
    e.step(warmup)
    c0 = e.counters()
    walk, stepms = e.bench_steps(steps, L2_FLUSH_BYTES, "both")
    c1 = e.counters()
    e.close()
    tot = float(stepms.sum()) / 1e3
    return {"workload": "C3: " + workloads.DESCRIPTIONS["c3"], "metric": "ant-steps/sec",
            "value": (c1.ant_steps - c0.ant_steps) / tot, "unit": "ant-steps/s",
            "ms_per_step": float(stepms.mean()), "walk_ms_per_step": float(walk.mean()),
            "iterations_timed": steps,
            "vehicle_routes_per_sec": (c1.vehicle_routes - c0.vehicle_routes) / tot,
            "kernel": "k_colony_grid (lattice walker, one-vehicle CTAs, 128 ants)"}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy bandwidth)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


REF_ALG_SHAPES = {"c1": (10, 10, "interior", 100), "c2": (32, 32, "all", 1000), "c3": (100, 100, "interior", 10000)}


def ref_algorithm_world(alg: str, config: str, seed: int = 1, max_steps: int = 5000):
    """(net, cfg) of a reference-algorithm run (dijkstra / aco / maco /
    maco-p; maco-p with preemptive signals, the others fixed, as
    harness.cpp:63-72) on a BASELINE grid config."""
    from paper_2010_14244_b200 import abi, networks
    if config not in REF_ALG_SHAPES:
        raise SystemExit(f"--algorithm {alg} runs on --config c1, c2 or c3")
    R, Cc, sig, V = REF_ALG_SHAPES[config]
    net = networks.grid(R, Cc, signals=sig)
    cfg = abi.default_config(algorithm=alg, vehicle_count=V, seed=seed, max_steps=max_steps)
    return net, cfg


def reference_algorithms_block(threads: int, alg: str = "maco-p", config: str = "c2", fold: bool = True):
    """SURVEY 8(d)(i)/(iii) on the GPU box, same process: the paper's own
    algorithm (MACO-P, preemptive signals) on C2 end to end through the C ABI
    -- gpu_run's path: gmaco_create with the engine's device SSSP building
    the exact distance table, gmaco_run, gmaco_collect -- against the
    reference's run() and parallel_run(nproc) (engine.cpp:435-450,
    parallel.cpp:276-291) including all_pairs_distances, which they need; and
    the F+G edge kernel (fold_maco_edge + evaporate_one) in edge-updates/s."""
    import torch
    from oracle import oracle as O
    from paper_2010_14244_b200 import abi
    from paper_2010_14244_b200.engine import Engine
    if not O.ref_available():
        return {"unavailable": "oracle/_ref not built"}
    net, cfg = ref_algorithm_world(alg, config)
    ours, runs, res = [], [], None
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e = Engine(net, cfg, abi.DistanceDesc(kind=abi.DIST_DENSE))  # device SSSP builds the table
        t1 = time.perf_counter()
        res = e.run()
        t2 = time.perf_counter()
        ctr = e.counters()
        e.close()
        ours.append(t2 - t0)
        runs.append(t2 - t1)
    ours_s, run_s = float(np.median(ours[1:])), float(np.median(runs[1:]))
    steps, decisions = int(res[0].steps_executed), int(ctr.decisions)
    seq, par, seq_run_ms, par_run_ms, ref = [], [], [], [], None
    for _ in range(3):
        t0 = time.perf_counter()
        ref = O.ref_run(net, cfg)
        seq.append(time.perf_counter() - t0)
        seq_run_ms.append(ref[0].wall_clock_ms)
        t0 = time.perf_counter()
        rp = O.ref_run(net, cfg, threads)
        par.append(time.perf_counter() - t0)
        par_run_ms.append(rp[0].wall_clock_ms)
    seq_s, par_s = float(np.median(seq)), float(np.median(par))
    R, Cc, sig, V = REF_ALG_SHAPES[config]
    block = {
        "workload": f"{config.upper()} network ({R}x{Cc}, {sig} intersections signalized), {V} vehicles, algorithm "
                    f"{alg} ({'preemptive' if alg == 'maco-p' else 'fixed'} signals; the reference's own path), "
                    "whole run to completion",
        "identical_to_reference": O.results_identical(res, ref),
        "steps": steps, "decisions": decisions,
        "ours": {"e2e_s": ours_s, "run_s": run_s, "steps_per_sec_e2e": steps / ours_s,
                 "decisions_per_sec_e2e": decisions / ours_s,
                 "includes": "gmaco_create from host arrays (device SSSP distance table) + gmaco_run + gmaco_collect"},
        "reference_run": {"e2e_s": seq_s, "run_ms": float(np.median(seq_run_ms)), "threads": 1,
                          "includes": "all_pairs_distances + run(cfg, dist)"},
        "reference_parallel_run": {"e2e_s": par_s, "run_ms": float(np.median(par_run_ms)), "threads": threads,
                                   "includes": f"all_pairs_distances + parallel_run(cfg, dist, {threads})"},
        "speedup_e2e_vs_run": seq_s / ours_s, "speedup_e2e_vs_parallel_run": par_s / ours_s,
        "speedup_run_only_vs_run": float(np.median(seq_run_ms)) / 1e3 / run_s,
    }
    if not fold:
        return block
    # (iii) F+G edge kernel: reference fold + evaporation on all host threads
    # over the C3 network with a step's worth of decisions, against this
    # engine's whole stage C..G tail (signals, motion, fold + evaporation) of
    # a C3 maco step, in edge-updates/s
    net3, cfg3 = ref_algorithm_world("maco", "c3")
    rng = np.random.default_rng(1)
    tau = rng.integers(0, 10 ** 8, net3.edge_count)
    e3 = Engine(net3, cfg3, net3.grid_distance())
    e3.step(5)
    walk, stepms = e3.bench_steps(20, L2_FLUSH_BYTES, "both")
    dpst = max(1, int(e3.counters().decisions / (25)))
    e3.close()
    dec = rng.integers(0, net3.edge_count, dpst)
    sec, _ = O.ref_fold_bench(tau, dec, 20, threads, cfg3.pheromone)
    tail_s = float((stepms - walk).mean()) / 1e3
    block["fold_edge_updates_per_sec"] = {
        "network": "C3 grid 100x100 (39,600 edges), maco (network-wide fold)",
        "reference": net3.edge_count * 20 / sec, "reference_threads": threads,
        "ours_tail": net3.edge_count / tail_s if tail_s > 0 else None,
        "ours_note": "whole cooperative tail per step (signals + motion + fold + evaporation), L2 flushed",
        "ours_step_ms": float(stepms.mean()), "ours_decide_ms": float(walk.mean()),
    }
    return block


# ----------------------------------------------------------------------------
# reference arm
# ----------------------------------------------------------------------------
def reference_world(seed, max_steps):
    from oracle import oracle as O
    from paper_2010_14244_b200 import abi, networks
    net = networks.grid(GRID, GRID, signals="all")
    cfg = abi.default_config(algorithm="aco", controller="preemptive", vehicle_count=VEHICLES, seed=seed,
                             max_steps=max_steps)
    return O.RefWorld(net, cfg), net


class RefSampler:
    """Reference colony iterations on a C2 world; a finished world is
    replaced by a fresh one (next seed) so no timed iteration is empty."""

    def __init__(self, threads):
        self.threads = threads
        self.seed = 1
        self.w = None

    def iteration(self):
        if self.w is None or self.w.finished():
            self.w, _ = reference_world(self.seed, 100000)
            self.seed += 1
        t0 = time.perf_counter()
        s, r = self.w.colony_iteration(ANTS, self.threads)
        return s, r, time.perf_counter() - t0


class RefStepSampler:
    """Reference-algorithm steps (sequential_step, engine.cpp:352-400) on the
    --config world; ant-steps = routing decisions (one next_node_* call
    each).  A finished world is replaced by a fresh one (next seed)."""

    def __init__(self, alg, config):
        self.alg, self.config, self.seed, self.w = alg, config, 1, None

    def iteration(self):
        from oracle import oracle as O
        if self.w is None or self.w.finished():
            net, cfg = ref_algorithm_world(self.alg, self.config, self.seed)
            self.w = O.RefWorld(net, cfg)
            self.seed += 1
        d0 = int(self.w.vehicles()["decisions"].sum())
        t0 = time.perf_counter()
        self.w.step(1)
        dt = time.perf_counter() - t0
        return int(self.w.vehicles()["decisions"].sum()) - d0, 0, dt


def run_reference(args, rank, world):
    if rank != 0:
        return
    from oracle import oracle as O
    if not O.ref_available():
        emit({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"})
        return
    if args.algorithm != "colony":
        smp = RefStepSampler(args.algorithm, args.config)
        for _ in range(args.warmup):
            smp.iteration()
        dec = 0
        dt = 0.0
        for _ in range(args.steps):
            d, _, t = smp.iteration()
            dec += d
            dt += t
        value = dec / dt
        emit({"impl": "reference", "metric": "ant-steps/sec", "value": value, "unit": "ant-steps/s",
              "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
              "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+int64",
              "data": "synthetic", "config": config_block(args, 1),
              "engine_steps_per_sec": args.steps / dt,
              "cpu_baseline": {"value": value, "unit": "ant-steps/s", "cores": 1, "kind": "reference",
                               "cpu_model": cpu_model(),
                               "sample": f"{args.steps} sequential_step calls of the reference ({args.algorithm}, "
                                         f"{args.config.upper()}; ant-step = one routing decision)"},
              "e2e": {"value": value, "unit": "ant-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
        return
    threads = os.cpu_count() or 1
    smp = RefSampler(threads)
    for _ in range(args.warmup):
        smp.iteration()
    steps = routes = 0
    dt = 0.0
    for _ in range(args.steps):
        s, r, t = smp.iteration()
        steps += s
        routes += r
        dt += t
    value = steps / dt
    line = {
        "impl": "reference", "metric": "ant-steps/sec", "value": value, "unit": "ant-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+int64",
        "data": "synthetic", "config": config_block(args, 1),
        "vehicle_routes_per_sec": routes / dt,
        "cpu_baseline": {"value": value, "unit": "ant-steps/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"{args.steps} colony iterations of the C2 workload, reference "
                                   f"next_node_aco tours on {threads} std::threads + sequential_step"},
        "e2e": {"value": value, "unit": "ant-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def cpu_baseline(seconds):
    """Bounded sample of the reference arm on this host (rank 0, N=1)."""
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    if O.ref_available():
        smp = RefSampler(threads)
        smp.iteration()
        steps = its = 0
        dt = 0.0
        while dt < seconds:
            s, _, t = smp.iteration()
            steps += s
            dt += t
            its += 1
        return {"value": steps / dt, "unit": "ant-steps/s", "cores": threads, "kind": "reference",
                "cpu_model": cpu_model(),
                "sample": f"{its} colony iterations (C2, 64 ants, reference next_node_aco on {threads} "
                          f"threads + sequential_step; finished worlds restarted), {dt:.1f} s"}
    from paper_2010_14244_b200 import networks
    net = networks.grid(GRID, GRID, signals="all")
    w = O.PortWorld(net, workload_config(1, 1000), net.grid_distance())
    t0 = time.perf_counter()
    its = 0
    while time.perf_counter() - t0 < seconds:
        w.step(1)
        its += 1
    dt = time.perf_counter() - t0
    return {"value": w.counters().ant_steps / dt, "unit": "ant-steps/s", "cores": 1, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{its} colony iterations of the C2 workload on the C oracle, {dt:.1f} s"}


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------
def make_engine(wl, local, rank, world, uid: bytes, max_steps=None):
    from paper_2010_14244_b200.engine import Engine
    net, cfg, dist, _keep = wl
    if max_steps is not None:
        cfg.max_steps = max_steps
    eng = Engine(net, cfg, dist, device=local)
    if uid:  # one world, vehicles sharded over the ranks; NCCL exchange inside the step graph
        eng.attach_comm(rank, world, uid)
    return eng


def build_workload(args, world):
    """(net, cfg, dist, keepalive) of --config.  C2 scales weakly (1,000
    vehicles' colonies per GPU); the larger configs keep their fleet and
    shard it (strong scaling), as BASELINE.json states them."""
    from paper_2010_14244_b200 import workloads
    max_steps = args.warmup + args.steps + 1
    if args.algorithm != "colony":
        net, cfg = ref_algorithm_world(args.algorithm, args.config, 1, max_steps=100000)
        return net, cfg, net.grid_distance(), None
    if args.config == "c2":
        return workloads.c2(seed=1, max_steps=max_steps, vehicles=VEHICLES * world)
    return workloads.CONFIGS[args.config](seed=1, max_steps=max_steps)


def rank_breakdown(me, dist, world, vehicles, net, cfg):
    """Per-rank timings gathered on rank 0: walk = stage B on the rank's
    shard; exchange_and_tail = the in-graph NCCL exchange (decision-record
    allgather + deposit allreduce) plus the replicated tail.
    exchange_probe_ms times the same two collectives alone through
    torch.distributed on the same sizes.  Diagnosis only: a failure here is
    recorded, never raised."""
    import torch
    from paper_2010_14244_b200 import abi
    try:
        P = -(-vehicles // world)
        dec = torch.zeros(P, dtype=torch.int32, device="cuda")
        gat = torch.zeros(P * world, dtype=torch.int32, device="cuda")
        dep = torch.zeros(net.edge_count, dtype=torch.int64, device="cuda")
        needs_dep = cfg.algorithm == abi.COLONY and cfg.colony.deposit == abi.DEPOSIT_BEST_TOUR
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        for it in range(13):
            if it == 3:
                torch.cuda.synchronize()
                dist.barrier()
                ev0.record()
            dist.all_gather_into_tensor(gat, dec)
            if needs_dep:
                dist.all_reduce(dep)
        ev1.record()
        torch.cuda.synchronize()
        me["exchange_probe_ms"] = ev0.elapsed_time(ev1) / 10
        ranks = [None] * world
        dist.all_gather_object(ranks, me)
        return ranks
    except Exception as exc:  # noqa: BLE001
        return [dict(me, breakdown_error=repr(exc))]


def run_ours(args, rank, world, local):
    import ctypes as C

    import torch
    from paper_2010_14244_b200 import abi, engine, networks

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    job_uid = []

    def fresh_uid():
        """The job's NCCL unique id, from rank 0.  Every engine of this run
        attaches with it; the library creates the communicator once (first
        attach, outside the e2e timing) and later engines share it."""
        if world == 1 and not args.force_comm:
            return b""
        if job_uid:
            return job_uid[0]
        box = [None]
        if rank == 0:
            buf = C.create_string_buffer(128)
            rc = engine.load().gmaco_nccl_unique_id(buf)
            assert rc == 0, "ncclGetUniqueId failed"
            box[0] = buf.raw
        if dist:
            dist.broadcast_object_list(box, src=0)
        job_uid.append(box[0])
        return box[0]
    wl = build_workload(args, world)
    net, cfg0 = wl[0], wl[1]
    vehicles = cfg0.vehicle_count

    # ---- device-resident throughput (value) ---------------------------------
    # K back-to-back iterations enqueued without host sync (one CUDA graph
    # each), each bracketed by exactly two CUDA events on the engine stream; a
    # 512 MiB memset flushes L2 before every iteration, outside the events.
    eng = make_engine(wl, local, rank, world, fresh_uid())
    eng.step(args.warmup)
    c0 = eng.counters()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    with ClockSampler(local) as clk:
        _, stepms = eng.bench_steps(args.steps, L2_FLUSH_BYTES, "step")
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    c1 = eng.counters()
    step_ms = float(stepms.sum())
    ant_steps = c1.ant_steps - c0.ant_steps
    routes = c1.vehicle_routes - c0.vehicle_routes
    alg_bytes = c1.walk_bytes - c0.walk_bytes
    kernels = c1.kernels_per_step
    eng.close()

    # walk kernel split (roofline): the same K iterations replayed on a fresh,
    # identically seeded engine (the run is deterministic), two events per
    # iteration around stage B only
    engw = make_engine(wl, local, rank, world, fresh_uid())
    engw.step(args.warmup)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    walk, _ = engw.bench_steps(args.steps, L2_FLUSH_BYTES, "walk")
    torch.cuda.synchronize()
    assert engw.counters().ant_steps == c1.ant_steps, "walk replay diverged from the timed run"
    engw.close()
    walk_ms = float(walk.sum())

    # chained (no flush, multi-step CUDA graphs), for reference
    chained_s, chained_steps = 1.0, 0
    if not args.skip_extra:
        eng2 = make_engine(wl, local, rank, world, fresh_uid())
        eng2.step(args.warmup)
        s0 = eng2.counters().ant_steps
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        eng2.step(args.steps)
        chained_s = time.perf_counter() - t0
        chained_steps = eng2.counters().ant_steps - s0
        eng2.close()

    # ---- end to end through the C ABI from host buffers (e2e) ---------------
    e2e_dt, e2e_steps, completed, e2e_phases = 1.0, 0, None, None
    h2d = net.edge_count * (4 + 4 + 8 + 4) + net.node_count * 1
    d2h = vehicles * 5
    if not args.skip_extra:
        uid = fresh_uid()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        e = make_engine(wl, local, rank, world, uid)  # H2D of all inputs
        # every step's vehicle states come back to host memory: double-buffered
        # (step k+1 is already enqueued while step k's snapshot is copied out)
        st = [np.zeros(vehicles, dtype=np.uint8) for _ in range(2)]
        oe = [np.zeros(vehicles, dtype=np.int32) for _ in range(2)]
        views = [abi.VehicleView(state=abi.ptr(st[i], C.c_uint8), on_edge=abi.ptr(oe[i], C.c_int32))
                 for i in range(2)]
        t1 = time.perf_counter()
        e.step(args.warmup)
        t2 = time.perf_counter()
        for k in range(args.steps):
            e.step_snapshot(views[k & 1], k & 1)  # one step + its state snapshot: one graph launch
            if k:
                e.vehicles_wait((k - 1) & 1, views[(k - 1) & 1])
        e.vehicles_wait((args.steps - 1) & 1, views[(args.steps - 1) & 1])
        t3 = time.perf_counter()
        res = e.collect()
        e2e_dt = time.perf_counter() - t0
        e2e_phases = {"create_ms": 1e3 * (t1 - t0), "warmup_ms": 1e3 * (t2 - t1),
                      "loop_us_per_step": 1e6 * (t3 - t2) / args.steps, "collect_ms": 1e3 * (e2e_dt - (t3 - t0))}
        e2e_steps = e.counters().ant_steps
        completed = res[0].completed_count
        e.close()

    # ---- per-rank breakdown (diagnosis of a scaling run) -------------------------
    me = {"rank": rank, "walk_ms": walk_ms / args.steps, "step_ms": step_ms / args.steps,
          "exchange_and_tail_ms": (step_ms - walk_ms) / args.steps, "ant_steps": ant_steps}
    ranks = rank_breakdown(me, dist, world, vehicles, net, cfg0) if dist and world > 1 else [me]

    # ---- reduce over ranks (time: max; work: sum) ------------------------------
    vals = torch.tensor([step_ms / 1e3, e2e_dt, chained_s, walk_ms], dtype=torch.float64, device="cuda")
    tot = torch.tensor([ant_steps, routes, e2e_steps, chained_steps], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    t_dev, e2e_dt, chained_s, _ = vals.tolist()
    tot_steps, tot_routes, tot_e2e, tot_chained = tot.tolist()
    if rank != 0:
        eng.close()
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_src = measured_peak()
    launches = args.steps
    walk_avg_s = (walk_ms / 1e3) / launches
    achieved = (alg_bytes / launches) / walk_avg_s / 1e9 if walk_avg_s > 0 else 0.0
    traffic, traffic_src = None, None
    try:  # DRAM bytes per walk launch from the committed ncu capture (profiles/)
        with open(os.path.join(ROOT, "profiles", "walk_traffic.json")) as f:
            rec = json.load(f)[args.config if args.algorithm == "colony" else f"{args.algorithm}-{args.config}"]
        traffic, traffic_src = rec["dram_bytes_per_launch"], rec["source"]
    except (OSError, KeyError, ValueError):
        pass
    lattice = args.config != "c4"
    walk_kernel = ("k_colony_grid (stage-B lattice colony walk)" if lattice else
                   "k_colony_qt (stage-B ant-queue colony walk over per-target candidate rows; "
                   "refresh/pro/epi kernels inside the timed walk)")
    if args.algorithm != "colony":
        walk_kernel = "k_decide (stage B: one next_node_* decision per vehicle at a node)"
    note = ("latency-bound: one colony iteration is a ~15 us dependent walk over L2/SMEM-resident state "
            "(~1 MB), see DESIGN.md §7" if args.config in ("c1", "c2") else
            "throughput-bound gather walk, see DESIGN.md §7")
    if args.algorithm == "colony" and args.config in ("c3", "c5"):
        note = ("frac is of the SURVEY 8(d) byte model, which counts every table read a walk makes; the lattice "
                "walker serves them from L1/L2 (real DRAM traffic per launch: 'traffic'), so frac > 1 is on-chip "
                "reuse, not HBM above its peak. The kernel's real limiter is in 'limiter' (ncu): issue and the "
                "dependent L1/L2 round trip per hop, see DESIGN.md §7")
    limiter = None
    try:  # the walk kernel's ncu limiter (committed capture of the same workload)
        cap = {"c2": "c2_walk", "c3": "c3_walk", "c5": "c5_walk", "c4": "c4_qt"}[args.config]
        with open(os.path.join(ROOT, "profiles", f"r02_ncu_{cap}.json")) as f:
            rep = json.load(f)
        rep = rep[0] if isinstance(rep, list) else rep
        limiter = {"source": f"profiles/r02_ncu_{cap}.json", "issue_active_pct": float(rep["issue_active_%"].split()[0]),
                   "l1_lsu_wavefronts_pct": float(rep["l1_lsu_wavefronts_%"].split()[0]),
                   "top_stalls_pct": dict(list(rep["stalls_%"].items())[:3]),
                   "dram_gbps": (traffic / walk_avg_s / 1e9) if (traffic and walk_avg_s > 0) else None}
    except (OSError, KeyError, ValueError, IndexError):
        pass
    line = {
        "metric": "ant-steps/sec",
        "value": tot_steps / t_dev,
        "unit": "ant-steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * t_dev / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64+int64",
        "data": "synthetic",
        "config": config_block(args, world, vehicles),
        "vehicle_routes_per_sec": tot_routes / t_dev,
        "engine_steps_per_sec": args.steps / t_dev,
        "ant_steps_per_iteration": tot_steps / args.steps,
        "walk_kernel_share": (walk_ms / step_ms) if step_ms else None,
        "chained_graph_value": tot_chained / chained_s,
        "ms_per_step_p50": float(np.median(stepms)),
        "walk_ms_per_step_p50": float(np.median(walk)),
        "gpu_launches": int(args.steps * kernels),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "traffic_source": traffic_src,
                     "kernel": walk_kernel,
                     "algorithmic_bytes_per_launch": alg_bytes / launches,
                     "algorithmic_bytes_model": "SURVEY 8(d): 8 + 4d + 4d(table dist) + 12c + 4(tour) per ant-step",
                     "avg_launch_us": walk_avg_s * 1e6,
                     "limiter": limiter if args.algorithm == "colony" else None,
                     "note": note},
        "e2e": {"value": tot_e2e / e2e_dt, "unit": "ant-steps/s",
                "h2d_bytes_per_step": h2d / (args.steps + args.warmup),
                "d2h_bytes_per_step": d2h,
                "includes": "gmaco_create from host arrays (H2D), warmup+timed steps, per-step D2H of "
                            "vehicle states (double-buffered: gmaco_step_snapshot/gmaco_vehicles_wait), gmaco_collect"
                            + ("; the job's NCCL communicator already exists (created once per job by its first "
                               "engine, outside this timing)" if job_uid else ""),
                "phases": e2e_phases},
        "clocks": clk.summary(),
        "per_rank": ranks,
        "completed_vehicles_e2e": completed,
    }
    headline = args.algorithm == "colony" and args.config == "c2"
    if world == 1 and not args.no_secondary and headline:
        line["secondary"] = secondary_c4(peak, peak_src)
        line["secondary_c3"] = secondary_c3()
    # the CPU-baseline leg (the only leg besides --impl reference that runs
    # the compiled reference, oracle/_ref): the reference's run() /
    # parallel_run() beside this engine's whole-run path, and the reference
    # colony workload for cpu_baseline
    if world == 1 and not args.no_secondary and not args.no_cpu_baseline and headline:
        line["reference_algorithms"] = reference_algorithms_block(os.cpu_count() or 1)
    if world == 1 and not args.no_cpu_baseline and headline:
        line["cpu_baseline"] = cpu_baseline(args.cpu_seconds)
    if world == 1 and not args.no_secondary and not args.no_cpu_baseline and args.algorithm != "colony" \
            and args.config in ("c1", "c2"):
        line["reference_run_comparison"] = reference_algorithms_block(os.cpu_count() or 1, args.algorithm,
                                                                      args.config, fold=False)
    if world == 1 and not args.no_cpu_baseline and args.algorithm != "colony":
        smp = RefStepSampler(args.algorithm, args.config)
        smp.iteration()
        dec, dt, its = 0, 0.0, 0
        while dt < args.cpu_seconds and its < 5000:
            d, _, t = smp.iteration()
            dec, dt, its = dec + d, dt + t, its + 1
        line["cpu_baseline"] = {"value": dec / dt, "unit": "ant-steps/s", "cores": 1, "kind": "reference",
                                "cpu_model": cpu_model(),
                                "sample": f"{its} reference sequential_step calls ({args.algorithm}, "
                                          f"{args.config.upper()}), {dt:.1f} s; ant-step = one routing decision"}
    eng.close()
    emit(line)
    if dist:
        dist.destroy_process_group()


def main():
    isolate_stdout()
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
