#!/usr/bin/env python
"""Benchmark: one Gauss-Newton / LM iteration of photometric BA at the
finest pyramid level (solve + pose update + linearise + assemble), the
metric of BASELINE.json ("GN iteration time (ms) and pixel-pair
residuals/sec at 1/2/4/8 B200; % HBM roofline").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4|c1|c2|c3|c5]
                  [--impl ours|reference]

value    = pixel-pair residuals per second of GN iteration, whole job
           (sum over pairs of depth-valid source pixels / iteration time),
           inputs resident in HBM.
e2e      = the same metric through the host-facing level session: every
           step copies the poses in from pinned host memory and reads the
           updated poses + cost back.
roofline = the linearisation kernel's algorithmic bytes (80 B per
           pixel-pair) / its CUDA-event time vs the measured
           HBM copy bandwidth of MEASURED_PEAKS.json.
cpu_baseline / --impl reference = the oracle C port of the reference path
           (oracle/, a test-infrastructure restatement of
           pkg/src/photoba/solver.py) on the host cores, on a bounded sample
           of pairs, extrapolated by pixel count, plus the full dense
           np.linalg.solve the reference performs.
Multi-GPU (torchrun): pairs are sharded, records gathered to rank 0,
poses broadcast; time = max over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BYTES_PER_PIXEL_PAIR = 80  # 5 fp64 cue values source + destination
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
CONFIGS = {
    "c1": dict(desc="synthetic RGB-D pinhole 10 frames 160x120, 1 level", kind="room", n=10,
               factors=(1,), max_translation=1.0),
    "c2": dict(desc="synthetic LiDAR spherical 64x1024 (HDL-64), 100 scans, 3 levels",
               kind="hdl64", n=100, spacing=0.1, factors=(4, 2, 1), max_translation=1.0),
    "c3": dict(desc="synthetic RGB-D pinhole 640x480 (TUM-shaped), 500 frames, 3 levels, "
                    "LM with block-Jacobi PCG", kind="tum", n=500, spacing=0.05,
               factors=(4, 2, 1), max_translation=1.0, solver="pcg"),
    "c4": dict(desc="synthetic OS0-128 128x1024, 1000 scans, 2 km corridor, 3 levels, ~20k pairs",
               kind="os0", n=1000, spacing=2.0, factors=(4, 2, 1), max_translation=40.0),
    "c5": dict(desc="joint LiDAR+RGB-D coupled BA: 500 platform poses x (OS0-128 128x1024 + "
                    "RGB-D 640x480), 3 levels", kind="fused", n=500, spacing=0.5,
               factors=(4, 2, 1), max_translation=10.0, max_translation_rgbd=1.0),
}

# pinhole camera looking along the corridor (+x of the platform): camera z ->
# platform x, camera x -> platform -y, camera y -> platform -z
FORWARD_CAMERA = np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])


def build_problem(name: str, device, n_override=None, normals: str = "estimate"):
    import torch

    import paper_2303_16878_b200 as P
    from paper_2303_16878_b200 import scenes as S

    c = CONFIGS[name]
    n = n_override or c["n"]
    graph_device = device if getattr(device, "type", "cpu") == "cuda" else None

    t_graph = 0.0

    def sensor_problem(cam, scene, gt, guess, ext, max_translation, sensor_id):
        nonlocal t_graph
        pyrs = S.device_pyramids(scene, cam, gt, ext, c["factors"], device, normals=normals)
        nodes = [P.FrameNode(k, guess[k], pyrs[k], 0.1 * k, sensor_id) for k in range(n)]
        crit = P.MatchCriteria(max_translation=max_translation)
        sensor_ext = P.SensorExtrinsics(ext)
        t0 = time.perf_counter()
        graph = P.build_graph(nodes, crit, extrinsics=sensor_ext, threads=8, device=graph_device)
        t_graph += time.perf_counter() - t0
        return P.BAProblem(graph, {sensor_id: sensor_ext})

    if c["kind"] in ("room", "hdl64", "os0", "tum"):
        if c["kind"] == "room":
            cam, scene, gt = S.rgbd_160(), S.BoxScene(), S.room_loop(n)
            ext = P.Pose.identity()
        elif c["kind"] == "tum":
            cam = S.tum_640()
            gt = S.corridor_trajectory(n, c["spacing"])
            scene = S.corridor_scene(c["spacing"] * n + 20.0)
            ext = P.Pose(FORWARD_CAMERA, [0.0, 0.0, 0.1])
        else:
            cam = S.hdl64() if c["kind"] == "hdl64" else S.lidar_os0_128()
            gt = S.corridor_trajectory(n, c["spacing"])
            scene = S.corridor_scene(c["spacing"] * n + 20.0)
            ext = P.Pose.identity() if c["kind"] == "hdl64" else P.Pose(np.eye(3), [0.0, 0.0, -0.05])
        guess = S.perturb(gt, 0.05, math.radians(2.0), 11)
        problems = [sensor_problem(cam, scene, gt, guess, ext, c["max_translation"], "sensor0")]
    else:  # fused: one platform trajectory, a LiDAR and a forward RGB-D camera
        cam = S.lidar_os0_128()
        gt = S.corridor_trajectory(n, c["spacing"])
        scene = S.corridor_scene(c["spacing"] * n + 20.0)
        guess = S.perturb(gt, 0.05, math.radians(2.0), 11)
        problems = [
            sensor_problem(cam, scene, gt, guess, P.Pose(np.eye(3), [0.0, 0.0, -0.05]),
                           c["max_translation"], "lidar0"),
            sensor_problem(S.tum_640(), scene, gt, guess, P.Pose(FORWARD_CAMERA, [0.1, 0.0, 0.1]),
                           c["max_translation_rgbd"], "rgbd0"),
        ]
    return problems, guess, gt, dict(name=name, desc=c["desc"], frames=n, cam=cam,
                                     level=len(c["factors"]) - 1, graph_seconds=t_graph)


def problems_pixel_pairs(problems, level) -> int:
    return sum(valid_pixel_pairs(p, level) for p in problems)


def valid_pixel_pairs(prob, level) -> int:
    """sum over pairs of depth-valid source pixels (solver.py:200-205)."""
    import torch

    counts = {}
    total = 0
    nodes = {n.id: n for n in prob.graph.nodes}
    for e in prob.graph.edges:
        cue = nodes[e.i].pyramid.levels[level]
        key = id(cue)
        if key not in counts:
            d = getattr(cue, "device_depth", None)
            cam = cue.intrinsics
            if d is not None:
                counts[key] = int(((d >= cam.depth_min) & (d <= cam.depth_max) & (d > 0)).sum())
            else:
                counts[key] = int(np.asarray(cue.depth_valid).sum())
        total += counts[key]
    return total


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class ClockSampler:
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
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback"


FLOPS_PER_VALID_PAIR = 1600  # SURVEY.md §8(d) F_alg, the reference formulation
FP64_PEAK_TFLOPS = 35.7       # DFMA, measured on this B200 by tools/micro/dmma.cu


def compute_roofline(counts, lin_ms):
    """Informational fp64 view of K1: algorithmic flops of the reference's
    formulation (F_alg per valid pixel-pair) over the measured DFMA peak.
    The q-basis executes fewer flops than F_alg, so this is an algorithmic
    rate, like roofline.achieved is for bytes."""
    if not counts or not lin_ms:
        return None
    valid = statistics.mean(counts)
    achieved = valid * FLOPS_PER_VALID_PAIR / (lin_ms * 1e-3) / 1e12
    return {"bound": "fp64", "unit": "TFLOP/s", "achieved": achieved,
            "peak": FP64_PEAK_TFLOPS, "peak_kind": "measured DFMA (tools/micro/dmma.cu)",
            "frac": achieved / FP64_PEAK_TFLOPS, "valid_pairs_per_launch": valid,
            "flops_per_valid_pair": FLOPS_PER_VALID_PAIR}


def ncu_traffic(name):
    """dram bytes per pixel-pair of the linearisation kernel from the committed
    ncu --set full summary (profiles/), scaled to this launch by the caller;
    None if absent or captured on another workload (it is a per-config
    figure: spherical c4 and pinhole c3 differ)."""
    p = ROOT / "profiles" / "linearize_traffic.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
    except Exception:
        return None
    return d if d.get("config", "c4") == name else None


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port on a bounded sample
# ---------------------------------------------------------------------------
def cpu_baseline(problems, guess, level, total_pp, target_seconds=12.0, threads=None):
    """The oracle C port on all host cores over a bounded prefix of every
    problem's pairs, extrapolated by pixel count, + the full dense LU solve."""
    import paper_2303_16878_b200 as P
    from oracle import oracle as O

    threads = threads or os.cpu_count() or 1
    cfg = P.SolverConfig()
    rows, _ = P.se3.pose_rows(guess)

    def sub_problem(prob, k):
        g = P.MatchGraph(prob.graph.nodes, prob.graph.edges[:k])
        return P.BAProblem(g, prob.extrinsics, prob.gauge_index)

    t_lin_total, parts = 0.0, []
    for prob in problems:
        budget = target_seconds / len(problems)
        # calibrate on a few pairs, then size the sample to the budget
        k = min(4, len(prob.graph.edges))
        lp = O.OracleLevel([sub_problem(prob, k)], level, cfg)
        t0 = time.perf_counter()
        lp.records(rows, True, threads)
        dt = max(time.perf_counter() - t0, 1e-6)
        per_pair = dt / k * min(k, threads) / threads if k < threads else dt / k
        k2 = int(max(k, min(len(prob.graph.edges), budget / max(per_pair, 1e-6))))
        k2 = max(min(threads, len(prob.graph.edges)), min(k2, len(prob.graph.edges)))
        lp = O.OracleLevel([sub_problem(prob, k2)], level, cfg)
        sample_pp = valid_pixel_pairs(sub_problem(prob, k2), level)
        t0 = time.perf_counter()
        lp.records(rows, True, threads)
        t_lin = time.perf_counter() - t0
        full_pp = valid_pixel_pairs(prob, level)
        t_lin_total += t_lin * (full_pp / max(sample_pp, 1))
        parts.append(f"the first {k2} of {len(prob.graph.edges)} pairs ({sample_pp} pixel-pairs, "
                     f"{t_lin:.2f} s)")
    # dense LU of the reference (np.linalg.solve on dim 6(N-1)), timed in full
    n = len(problems[0].graph.nodes)
    dim = 6 * (n - 1)
    rng = np.random.default_rng(0)
    A = rng.normal(size=(dim, 64))
    H = A @ A.T + np.eye(dim)
    b = rng.normal(size=dim)
    t0 = time.perf_counter()
    np.linalg.solve(H + 1e-3 * np.diag(np.diag(H)), -b)
    t_solve = time.perf_counter() - t0
    gens = np.zeros(n, np.int64)
    t0 = time.perf_counter()
    lp.apply_step(rows, gens, np.zeros(dim))
    t_upd = time.perf_counter() - t0
    t_iter = t_lin_total + t_solve + t_upd
    # one-thread rate on a small sample (BASELINE.md asks for T = 1 and T = all)
    prob0 = problems[0]
    k1 = min(2, len(prob0.graph.edges))
    lp1 = O.OracleLevel([sub_problem(prob0, k1)], level, cfg)
    pp1 = valid_pixel_pairs(sub_problem(prob0, k1), level)
    t0 = time.perf_counter()
    lp1.records(rows, True, 1)
    per_px_1 = (time.perf_counter() - t0) / max(pp1, 1)
    t_iter_1 = per_px_1 * total_pp + t_solve + t_upd
    return {
        "value": total_pp / t_iter,
        "unit": "pixel-pairs/s",
        "cores": threads,
        "kind": "port",
        "sample": (f"oracle C port (OpenMP {threads} threads) linearising " + "; ".join(parts) +
                   f", extrapolated by pixel count to {total_pp}; + full np.linalg.solve dim "
                   f"{dim} ({t_solve:.2f} s) + apply_step ({t_upd * 1e3:.1f} ms)"),
        "gn_iteration_ms_extrapolated": t_iter * 1e3,
        "value_1_thread": total_pp / t_iter_1,
        "sample_1_thread": f"first {k1} pairs ({pp1} pixel-pairs) on one thread, extrapolated",
    }


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2303_16878_b200 as P
    from paper_2303_16878_b200 import distributed as D
    from paper_2303_16878_b200 import native
    from paper_2303_16878_b200.device import DeviceLevel, FrameStore

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    if world > 1 or os.environ.get("PBA_FORCE_SHARDED") == "1":
        dist.init_process_group("nccl", device_id=device)
    lib = native.load()

    t_setup = time.perf_counter()
    problems, guess, gt, meta = build_problem(args.config, device, args.frames)
    if len(problems) > 1 and (world > 1 or os.environ.get("PBA_FORCE_SHARDED") == "1"):
        raise SystemExit("fused (multi-sensor) configs are benchmarked on one GPU")
    level = meta["level"]
    solver = args.solver or CONFIGS[args.config].get("solver", "cholesky")
    cfg = P.SolverConfig(linear_solver=solver)
    store = FrameStore(device)
    group = D.current_group()
    backend = D.make_level(problems, level, cfg, store, group)
    local_level = backend.local if hasattr(backend, "local") else backend
    rows, gens = P.se3.pose_rows(guess)
    backend.set_poses(rows, gens)
    cost0, count0 = backend.evaluate_current()
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    total_pp = problems_pixel_pairs(problems, level)
    n_pairs = sum(len(p.graph.edges) for p in problems)

    lam = cfg.lm_initial_lambda
    state = {"cost": cost0, "lam": lam}

    counts = []  # valid pixel-pairs (the reference's `count`) of every linearisation

    def step():
        ok_s, ok_u, c, n = backend.try_step(state["lam"])
        counts.append(n)
        if ok_s and ok_u and c < state["cost"] and n > 0:
            backend.accept()
            state["cost"] = c
            state["lam"] = max(state["lam"] * 0.5, 1e-12)
        else:
            state["lam"] *= cfg.lm_factor

    for _ in range(args.warmup):
        step()
    # LM state at the start of the timed region, restored before the e2e loop
    # so both loops run the identical sequence of steps
    snap_rows = local_level.poses[local_level.cur].cpu().numpy().copy()
    snap_gens = local_level.gens[local_level.cur].cpu().numpy().copy()
    snap_state = dict(state)
    stream = torch.cuda.current_stream(device)
    local_level.kernel_events = []
    if getattr(local_level, "has_solver", False):
        local_level.solve_events = []
    launches0 = lib.pba_kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed_ms = e0.elapsed_time(e1)
    launches = (lib.pba_kernel_launches() - launches0) / args.steps
    lin_ms = [a.elapsed_time(b) for a, b in local_level.kernel_events]
    solve_ms = [a.elapsed_time(b) for a, b in (local_level.solve_events or [])]
    local_level.kernel_events = None
    local_level.solve_events = None
    pcg_info = None
    if getattr(local_level, "pcg", False):
        it, relres, conv = local_level.pcg_info.cpu().tolist()
        pcg_info = {"iterations": int(it), "rel_residual": relres, "converged": bool(conv)}
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps

    # ---- e2e: host pose buffers in, poses + cost out, every step --------
    # Same start state and hence the same step sequence as the timed loop.
    # The step's input (current poses + generations) is copied in from pinned
    # host memory and its result (the accepted poses) copied back out, so the
    # next step starts from host data; cost/count/status come back inside
    # try_step's scalar readback.
    L = local_level
    backend.set_poses(snap_rows, snap_gens)
    backend.evaluate_current()
    state.update(snap_state)
    host_in = torch.from_numpy(snap_rows.copy()).pin_memory()
    gens_in = torch.from_numpy(snap_gens.copy()).pin_memory()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        L.poses[L.cur].copy_(host_in, non_blocking=True)
        L.gens[L.cur].copy_(gens_in, non_blocking=True)
        step()
        host_in.copy_(L.poses[L.cur], non_blocking=True)
        gens_in.copy_(L.gens[L.cur], non_blocking=True)
        stream.synchronize()
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / args.steps
    t = torch.tensor([e2e_ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())
    e2e = {"value": total_pp / (e2e_ms / 1e3), "unit": "pixel-pairs/s",
           "h2d_bytes_per_step": int(host_in.numel() * 8 + gens_in.numel() * 4),
           "d2h_bytes_per_step": int(host_in.numel() * 8 + gens_in.numel() * 4 + 64),
           "ms_per_step": e2e_ms,
           "path": "DeviceLevel.try_step via the C ABI; poses in/out through pinned host buffers"}

    if rank != 0:
        if dist.is_initialized():
            dist.destroy_process_group()
        return None

    peak, peak_kind = measured_peak_hbm()
    lin_avg_ms = statistics.mean(lin_ms) if lin_ms else float("nan")
    my_pp = getattr(local_level, "pixels_shard", None)
    shard_pp = total_pp if world == 1 else valid_pixel_pairs_shard(problems[0], level, local_level)
    achieved = shard_pp * BYTES_PER_PIXEL_PAIR / (lin_avg_ms / 1e3) / 1e9
    trafficd = ncu_traffic(args.config)
    traffic = None
    if trafficd and trafficd.get("dram_bytes_per_pixel_pair"):
        traffic = trafficd["dram_bytes_per_pixel_pair"] * shard_pp
    line = {
        "metric": "GN iteration throughput: pixel-pair residuals/s (one LM iteration at the "
                  "finest level: solve + pose update + linearise + assemble)",
        "value": total_pp / (ms_per_step / 1e3),
        "unit": "pixel-pairs/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {
            "workload": f"{args.config}: {meta['desc']}",
            "frames": meta["frames"],
            "pairs": n_pairs,
            "pixel_pairs_per_iteration": total_pp,
            "level": f"finest ({meta['cam'].height}x{meta['cam'].width})",
            "parallelism": f"pair-sharded x{world}" if world > 1 else "single GPU",
            "l2": "inputs larger than L2: %.1f GB of resident texels" % (store.texel_bytes() / 1e9),
            "precision": "fp64 throughout (geometry, residuals, Jacobians, H/b/cost sums)",
            "gn_iteration_ms": ms_per_step,
            "linear_solver": solver,
            "setup_seconds": round(t_setup, 2),
            "graph_seconds": round(meta["graph_seconds"], 2),
            "initial_cost": cost0,
            "initial_valid_blocks": count0,
        },
        "roofline": {
            "bound": "hbm",
            "kernel": "linearize_kernel (+ per-pair chunk reduce) via pba_linearize",
            "achieved": achieved,
            "peak": peak,
            "peak_kind": peak_kind,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": traffic,
            "linearize_ms": lin_avg_ms,
            "linearize_share_of_step": lin_avg_ms / ms_per_step,
            "solve_ms": statistics.mean(solve_ms) if solve_ms else None,
            "pcg_last_solve": pcg_info,
            "algorithmic_bytes_per_launch": shard_pp * BYTES_PER_PIXEL_PAIR,
        },
        "compute": compute_roofline(counts[args.warmup:args.warmup + args.steps], lin_avg_ms)
        if world == 1 else None,
        "e2e": e2e,
        "gpu_launches": int(round(launches)),
        "clocks": clocks.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(problems, guess, level, total_pp)
    print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()
    return line


def valid_pixel_pairs_shard(prob, level, local_level):
    import paper_2303_16878_b200 as P

    lo, hi = local_level.pair_lo, local_level.pair_hi
    g = P.MatchGraph(prob.graph.nodes, prob.graph.edges[lo:hi])
    return valid_pixel_pairs(P.BAProblem(g, prob.extrinsics, prob.gauge_index), level)


# ---------------------------------------------------------------------------
# reference arm: the oracle port on the host cores (rank 0 only)
# ---------------------------------------------------------------------------
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import torch

    device = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    problems, guess, gt, meta = build_problem(args.config, device, args.frames)
    level = meta["level"]
    total_pp = problems_pixel_pairs(problems, level)
    vals = []
    for k in range(args.warmup + args.steps):
        cb = cpu_baseline(problems, guess, level, total_pp, target_seconds=args.ref_seconds)
        if k >= args.warmup:
            vals.append(cb)
    v = statistics.median(c["value"] for c in vals)
    ms = statistics.median(c["gn_iteration_ms_extrapolated"] for c in vals)
    line = {
        "impl": "reference",
        "metric": "GN iteration throughput: pixel-pair residuals/s (one LM iteration at the "
                  "finest level: solve + pose update + linearise + assemble)",
        "value": v,
        "unit": "pixel-pairs/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {meta['desc']}", "frames": meta["frames"],
                   "pairs": sum(len(p.graph.edges) for p in problems),
                   "pixel_pairs_per_iteration": total_pp},
        "cpu_baseline": {"value": v, "unit": "pixel-pairs/s", "cores": vals[-1]["cores"],
                         "kind": "port", "sample": vals[-1]["sample"]},
        "e2e": {"value": v, "unit": "pixel-pairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--frames", type=int, default=None, help="override the frame count")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--solver", default=None, choices=["cholesky", "pcg"],
                    help="damped-system solver (default: pcg for c3, cholesky otherwise)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=4.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
