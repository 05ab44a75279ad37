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

METRIC = ("GN iteration throughput: pixel-pair residuals/s (one LM iteration at the finest "
          "level: solve + pose update + linearise + assemble)")
BYTES_PER_PIXEL_PAIR = 80  # 5 fp64 cue values source + destination
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
CONFIGS = {
    "c1": dict(desc="synthetic RGB-D pinhole 10 frames 160x120, 1 level", kind="room", n=10,
               factors=(1,), max_translation=1.0, pairs=24, pixel_pairs=460_800,
               sample_frames=10),
    "c2": dict(desc="synthetic LiDAR spherical 64x1024 (HDL-64), 100 scans, 3 levels",
               kind="hdl64", n=100, spacing=0.1, factors=(4, 2, 1), max_translation=1.0,
               pairs=722, pixel_pairs=47_316_992, sample_frames=100),
    "c3": dict(desc="synthetic RGB-D pinhole 640x480 (TUM-shaped), 500 frames, 3 levels, "
                    "LM with block-Jacobi PCG", kind="tum", n=500, spacing=0.05,
               factors=(4, 2, 1), max_translation=1.0, solver="pcg", pairs=6212,
               pixel_pairs=1_684_654_459, sample_frames=24),
    "c4": dict(desc="synthetic OS0-128 128x1024, 1000 scans, 2 km corridor, 3 levels, ~20k pairs",
               kind="os0", n=1000, spacing=2.0, factors=(4, 2, 1), max_translation=40.0,
               pairs=19258, pixel_pairs=2_519_907_096, sample_frames=48),
    "c5": dict(desc="joint LiDAR+RGB-D coupled BA: 500 platform poses x (OS0-128 128x1024 + "
                    "RGB-D 640x480), 3 levels", kind="fused", n=500, spacing=0.5,
               factors=(4, 2, 1), max_translation=10.0, max_translation_rgbd=1.0, pairs=10170,
               pixel_pairs=1_427_480_623, sample_frames=20),
}
# `pairs` / `pixel_pairs`: edge count and sum of depth-valid source pixels at
# the finest level of each full problem, as the GPU arm measures them live
# (round-1 bench lines, profiles/r01_bench_c*.json; test_c4_full_size_properties
# re-checks c4).  The reference arm never builds the full problem — it
# times a host-built prefix of `sample_frames` frames — so it quotes these.


L2_BYTES = 126 * 2 ** 20  # B200 L2


def l2_note(store) -> str:
    b = store.texel_bytes()
    if b > L2_BYTES:
        return "inputs larger than L2: %.1f GB of resident texels" % (b / 1e9)
    return "inputs fit in L2: %.1f MB of resident texels (not flushed between steps)" % (b / 1e6)


def workload_config(name: str, cam, frames: int, pairs: int, pixel_pairs: int, solver: str) -> dict:
    """The `config` object of the bench line; both arms emit exactly this."""
    c = CONFIGS[name]
    return {"workload": f"{name}: {c['desc']}", "frames": frames, "pairs": pairs,
            "pixel_pairs_per_iteration": pixel_pairs,
            "level": f"finest ({cam.height}x{cam.width})", "linear_solver": solver,
            "data": ("synthetic box-room renders (seeded), inputs fit in L2 (25 MB of texels; "
                     "the reference's own small case, not flushed between steps)"
                     if c["kind"] == "room" else
                     "synthetic box-corridor renders (seeded), inputs larger than L2")}

# pinhole camera looking along the corridor (+x of the platform): camera z ->
# platform x, camera x -> platform -y, camera y -> platform -z
FORWARD_CAMERA = np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])


def host_pyramids_estimated(scene, cam, platform_poses, ext, factors, threads):
    """Host-only pyramids (no GPU, no libpba_b200): torch-CPU renders, then
    the numpy pyramid builder (estimate_normals + downscale, bit-exact to the
    reference's build_pyramid, cues.py:342-375) on a thread pool."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_2303_16878_b200 import cueimage
    from paper_2303_16878_b200 import scenes as S

    rows = S.sensor_rows(platform_poses, ext)
    scales = tuple(1.0 / f for f in factors)
    inten, depth, _ = S.render_batch(scene, cam, rows)
    inten, depth = inten.numpy(), depth.numpy()
    with ThreadPoolExecutor(max_workers=max(1, threads)) as pool:
        return list(pool.map(lambda b: cueimage.build_pyramid(inten[b], depth[b], cam, scales),
                             range(rows.shape[0])))


def build_problem(name: str, device, n_override=None, normals: str = "estimate",
                  host: bool = False, prefix: int | None = None, threads: int = 8):
    """The App. C problem of config `name`.  Default: frames rendered and
    pyramids built on `device` (K6), graph built with K5.  host=True builds
    everything on the CPU without the product library (the reference arm);
    `prefix` keeps only the first `prefix` frames of the full trajectory
    (same scene, same seeded perturbation), whose edges are exactly the full
    edge list's pairs among those frames."""
    import torch

    import paper_2303_16878_b200 as P
    from paper_2303_16878_b200 import scenes as S

    c = CONFIGS[name]
    n_full = n_override or c["n"]
    n = min(prefix, n_full) if prefix else n_full
    graph_device = device if (not host and getattr(device, "type", "cpu") == "cuda") else None

    t_graph = 0.0

    def sensor_problem(cam, scene, gt, guess, ext, max_translation, sensor_id):
        nonlocal t_graph
        gt, guess = gt[:n], guess[:n]
        if host:
            pyrs = host_pyramids_estimated(scene, cam, gt, ext, c["factors"], threads)
        else:
            pyrs = S.device_pyramids(scene, cam, gt, ext, c["factors"], device, normals=normals)
        nodes = [P.FrameNode(k, guess[k], pyrs[k], 0.1 * k, sensor_id) for k in range(n)]
        crit = P.MatchCriteria(max_translation=max_translation)
        sensor_ext = P.SensorExtrinsics(ext)
        t0 = time.perf_counter()
        graph = P.build_graph(nodes, crit, extrinsics=sensor_ext, threads=threads, device=graph_device)
        t_graph += time.perf_counter() - t0
        return P.BAProblem(graph, {sensor_id: sensor_ext})

    if c["kind"] in ("room", "hdl64", "os0", "tum"):
        if c["kind"] == "room":
            cam, scene, gt = S.rgbd_160(), S.BoxScene(), S.room_loop(n_full)
            ext = P.Pose.identity()
        elif c["kind"] == "tum":
            cam = S.tum_640()
            gt = S.corridor_trajectory(n_full, c["spacing"])
            scene = S.corridor_scene(c["spacing"] * n_full + 20.0)
            ext = P.Pose(FORWARD_CAMERA, [0.0, 0.0, 0.1])
        else:
            cam = S.hdl64() if c["kind"] == "hdl64" else S.lidar_os0_128()
            gt = S.corridor_trajectory(n_full, c["spacing"])
            scene = S.corridor_scene(c["spacing"] * n_full + 20.0)
            ext = P.Pose.identity() if c["kind"] == "hdl64" else P.Pose(np.eye(3), [0.0, 0.0, -0.05])
        guess = S.perturb(gt, 0.05, math.radians(2.0), 11)
        problems = [sensor_problem(cam, scene, gt, guess, ext, c["max_translation"], "sensor0")]
    else:  # fused: one platform trajectory, a LiDAR and a forward RGB-D camera
        cam = S.lidar_os0_128()
        gt = S.corridor_trajectory(n_full, c["spacing"])
        scene = S.corridor_scene(c["spacing"] * n_full + 20.0)
        guess = S.perturb(gt, 0.05, math.radians(2.0), 11)
        problems = [
            sensor_problem(cam, scene, gt, guess, P.Pose(np.eye(3), [0.0, 0.0, -0.05]),
                           c["max_translation"], "lidar0"),
            sensor_problem(S.tum_640(), scene, gt, guess, P.Pose(FORWARD_CAMERA, [0.1, 0.0, 0.1]),
                           c["max_translation_rgbd"], "rgbd0"),
        ]
    return problems, guess[:n], gt[:n], dict(name=name, desc=c["desc"], frames=n, cam=cam,
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
    out = {"bound": "fp64", "unit": "TFLOP/s", "achieved": achieved,
           "kind": "algorithmic: F_alg (the reference formulation's flops per valid pixel-pair) "
                   "x valid pixel-pairs / K1 time; the q-basis kernel executes fewer flops, so "
                   "this is not an executed rate",
           "peak": FP64_PEAK_TFLOPS, "peak_kind": "measured DFMA (tools/micro/dmma.cu)",
           "frac": achieved / FP64_PEAK_TFLOPS, "valid_pairs_per_launch": valid,
           "flops_per_valid_pair": FLOPS_PER_VALID_PAIR}
    # the executed fp64 utilisation of the same kernel, from the committed ncu capture
    p = ROOT / "profiles" / "linearize_traffic.json"
    try:
        d = json.loads(p.read_text())
        if d.get("fp64_pipe_active_pct") is not None:
            out["ncu_fp64_pipe_active_pct"] = d["fp64_pipe_active_pct"]
            out["ncu_issue_active_pct"] = d.get("issue_active_pct")
            out["ncu_source"] = d.get("source")
    except Exception:
        pass
    return out


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
# CPU baseline / reference arm: the oracle port on a host-built sample
# ---------------------------------------------------------------------------
class ReferenceSample:
    """A bounded sample of config `name` for the reference CPU path, built
    entirely on the host (torch-CPU renders, numpy pyramids, host
    build_graph; libpba_b200 is never loaded): the first `sample_frames`
    frames of the full trajectory, whose edges are the full edge list's pairs
    among them.  One step = what the reference does per LM iteration
    (solver.py:505-537): linearise every sampled pair with the oracle C port
    on all host cores (PairContext.evaluate + _edge_term), assemble them
    densely in edge order (solver.py:428-449), solve the damped dense system
    of the FULL dimension 6(N-1) with np.linalg.solve (solver.py:510-512) and
    apply the step to all N poses (solver.py:451-460).  The full-iteration
    time is extrapolated from the sample by pixel count (linearisation) and
    pair count (assembly); c1 and c2 are sampled whole (no extrapolation)."""

    def __init__(self, name: str, frames: int | None = None, threads: int | None = None):
        import paper_2303_16878_b200 as P
        from oracle import oracle as O

        c = CONFIGS[name]
        self.name = name
        self.threads = threads or os.cpu_count() or 1
        n_full = frames or c["n"]
        m = min(c["sample_frames"], n_full)
        t0 = time.perf_counter()
        problems, guess, _, meta = build_problem(name, None, n_full, host=True, prefix=m,
                                                 threads=self.threads)
        self.setup_seconds = time.perf_counter() - t0
        self.level = meta["level"]
        self.cam = meta["cam"]
        self.cfg = P.SolverConfig()
        self.rows, _ = P.se3.pose_rows(guess)
        self.lp = O.OracleLevel(problems, self.level, self.cfg)
        self.sample_frames = m
        self.sample_pairs = sum(len(p.graph.edges) for p in problems)
        self.sample_pp = problems_pixel_pairs(problems, self.level)
        full = n_full == c["n"]
        self.n_full = n_full
        self.full_pairs = c["pairs"] if full else None
        self.full_pp = c["pixel_pairs"] if full else None
        if m == n_full:  # sampled whole
            self.full_pairs, self.full_pp = self.sample_pairs, self.sample_pp
        dim = 6 * (n_full - 1)
        rng = np.random.default_rng(0)
        A = rng.normal(size=(dim, 64))
        self.H = A @ A.T + np.eye(dim)  # SPD stand-in of the assembled H (LU cost is data-independent)
        self.b = rng.normal(size=dim)
        reps = -(-n_full // m)
        self.full_rows = np.ascontiguousarray(np.tile(self.rows, (reps, 1))[:n_full])
        self.full_gens = np.zeros(n_full, np.int64)

    def extrapolate(self, full_pairs, full_pp):
        self.full_pairs, self.full_pp = full_pairs, full_pp

    def step(self):
        """One reference LM iteration on the sample; returns the timings (s)."""
        from oracle import oracle as O

        t0 = time.perf_counter()
        recs = self.lp.records(self.rows, True, self.threads)
        t1 = time.perf_counter()
        self.lp.assemble(recs)
        t2 = time.perf_counter()
        lam = self.cfg.lm_initial_lambda
        delta = np.linalg.solve(self.H + lam * np.diag(np.diag(self.H)), -self.b)
        t3 = time.perf_counter()
        O.apply_step(self.full_rows, self.full_gens, 1e-9 * delta, 0)
        t4 = time.perf_counter()
        return {"lin": t1 - t0, "asm": t2 - t1, "solve": t3 - t2, "update": t4 - t3,
                "wall": t4 - t0}

    def iteration_seconds(self, t) -> float:
        """Full-problem LM iteration time extrapolated from one sample step."""
        return (t["lin"] * self.full_pp / max(self.sample_pp, 1)
                + t["asm"] * self.full_pairs / max(self.sample_pairs, 1)
                + t["solve"] + t["update"])

    def one_thread_rate(self) -> tuple:
        """Linearisation rate of one thread over the first two pairs."""
        k = min(2, len(self.lp.pairs))
        t0 = time.perf_counter()
        self.lp.records(self.rows, True, 1, pair_subset=list(range(k)))
        dt = time.perf_counter() - t0
        pp = sum(self._pair_pixels(p) for p in range(k))
        return pp / max(dt, 1e-9), f"first {k} pairs ({pp} pixel-pairs) on one thread"

    def _pair_pixels(self, p) -> int:
        src = self.lp.images[self.lp.pairs[p][2]]
        return int(np.asarray(src.depth_valid).sum())

    def describe(self, t) -> str:
        ext = ("" if self.sample_pp == self.full_pp else
               f", extrapolated by pixel count to {self.full_pp} ({self.full_pairs} pairs)")
        return (f"oracle C port (OpenMP {self.threads} threads): host-built first "
                f"{self.sample_frames} of {self.n_full} frames, {self.sample_pairs} pairs, "
                f"{self.sample_pp} pixel-pairs linearised in {t['lin']:.2f} s + dense assembly "
                f"{t['asm'] * 1e3:.1f} ms{ext}; + np.linalg.solve dim {6 * (self.n_full - 1)} "
                f"({t['solve']:.2f} s) + apply_step of {self.n_full} poses "
                f"({t['update'] * 1e3:.1f} ms)")


def cpu_baseline(name, frames, full_pairs, full_pp):
    """cpu_baseline object of the GPU arm's line: one warm sample step."""
    smp = ReferenceSample(name, frames)
    smp.extrapolate(full_pairs, full_pp)
    smp.step()
    t = smp.step()
    it = smp.iteration_seconds(t)
    rate1, desc1 = smp.one_thread_rate()
    lin_full_1 = full_pp / rate1
    it1 = (lin_full_1 + t["asm"] * full_pairs / max(smp.sample_pairs, 1) + t["solve"]
           + t["update"])
    return {"value": full_pp / it, "unit": "pixel-pairs/s", "cores": smp.threads, "kind": "port",
            "linearize_rate": smp.sample_pp / t["lin"], "solve_seconds": t["solve"],
            "sample": smp.describe(t), "gn_iteration_ms_extrapolated": it * 1e3,
            "value_1_thread": full_pp / it1, "sample_1_thread": desc1 + ", extrapolated"}


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
    # Small problems on one GPU run the LM level as one conditional-graph
    # launch (DeviceLevel.lm_level_device, the path solve_hierarchical takes
    # there); the timed region is then one launch of exactly --steps
    # iterations (no termination test, unbounded lambda) instead of
    # --steps host-driven graph replays.
    use_loop = (world == 1 and args.lm_loop != "host"
                and getattr(backend, "lm_loop_ready", lambda: False)())
    if use_loop:
        return run_ours_device_loop(args, backend, lib, problems, level, meta, cfg, solver,
                                    store, state, counts, t_setup, cost0, count0, total_pp,
                                    n_pairs, device)
    if hasattr(backend, "prepare_graphs"):
        backend.prepare_graphs()  # single GPU: the step is a CUDA graph replay from here on
    # LM state at the start of the timed region, restored before the e2e loop
    # so both loops run the identical sequence of steps
    snap_rows = local_level.poses[local_level.cur].cpu().numpy().copy()
    snap_gens = local_level.gens[local_level.cur].cpu().numpy().copy()
    snap_state = dict(state)
    stream = torch.cuda.current_stream(device)
    local_level.kernel_events = []
    if getattr(local_level, "has_solver", False):
        local_level.solve_events = []
    launches0 = lib.pba_kernel_launches() + getattr(local_level, "graph_launches_replayed", 0)
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
    launches = (lib.pba_kernel_launches() + getattr(local_level, "graph_launches_replayed", 0)
                - launches0) / args.steps
    def _ms(x):  # graph replays log floats, eager steps (start, stop) event pairs
        return x if isinstance(x, float) else x[0].elapsed_time(x[1])

    lin_ms = [_ms(x) for x in local_level.kernel_events]
    solve_ms = [_ms(x) for x in (local_level.solve_events or [])]
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
    shard_pp = total_pp if world == 1 else valid_pixel_pairs_shard(problems, level, local_level)
    achieved = shard_pp * BYTES_PER_PIXEL_PAIR / (lin_avg_ms / 1e3) / 1e9
    trafficd = ncu_traffic(args.config)
    traffic = None
    if trafficd and trafficd.get("dram_bytes_per_pixel_pair"):
        traffic = trafficd["dram_bytes_per_pixel_pair"] * shard_pp
    line = {
        "metric": METRIC,
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
        "config": workload_config(args.config, meta["cam"], meta["frames"], n_pairs, total_pp,
                                  solver),
        "parallelism": f"pair-sharded x{world}" if world > 1 else "single GPU",
        "setup": {
            "l2": l2_note(store),
            "precision": "fp64 throughout (geometry, residuals, Jacobians, H/b/cost sums)",
            "gn_iteration_ms": ms_per_step,
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
        # the reference's `count` (valid blocks) per second too
        "valid_blocks_per_s": (statistics.mean(counts[args.warmup:args.warmup + args.steps])
                               / (ms_per_step / 1e3)) if counts else None,
        "gpu_launches": int(round(launches)),
        "clocks": clocks.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, args.frames, n_pairs, total_pp)
    if world == 1 and not args.no_e2e_api:
        cb = line.get("cpu_baseline") or {}
        line["e2e_api"] = e2e_api(args.config, args.frames, device, cb.get("linearize_rate"),
                                  cb.get("solve_seconds"))
    print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()
    return line


class _NoTermination:
    """LM settings of the bench's device loop: the reference's lambda factor,
    no relative-decrease stop, so exactly --steps iterations run."""
    lm_factor = 10.0
    termination_rel_decrease = -1.0


def run_ours_device_loop(args, lv, lib, problems, level, meta, cfg, solver, store, state, counts,
                         t_setup, cost0, count0, total_pp, n_pairs, device):
    """The timed loop as one device-resident LM launch (single GPU, small
    problems).  Kernel times for the roofline come from eager launches of the
    same linearisation and solve at the end state (the loop body holds no
    timing events); e2e adds the host pose upload, the initial evaluation and
    the pose / record readback of the API call, per iteration."""
    import torch

    import paper_2303_16878_b200 as P

    assert cfg.lm_factor == _NoTermination.lm_factor
    stream = torch.cuda.current_stream(device)
    cost, count = lv.evaluate_current()
    lv.lm_level_device(cost, count, state["lam"], _NoTermination, 2, float("inf"))  # warm
    snap_rows, snap_gens = lv.current_rows()
    cost, count = lv.evaluate_current()
    lam = state["lam"]
    launches0 = lib.pba_kernel_launches() + lv.graph_launches_replayed
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(device.index or 0) as clocks:
        recs, err, _, _ = lv.lm_level_device(cost, count, lam, _NoTermination, args.steps,
                                             float("inf"), details=True, events=(e0, e1))
        torch.cuda.synchronize()
    elapsed_ms = e0.elapsed_time(e1)
    if err or len(recs) != args.steps:
        raise RuntimeError(f"device LM loop ran {len(recs)} of {args.steps} iterations "
                           f"(error {err})")
    launches = (lib.pba_kernel_launches() + lv.graph_launches_replayed - launches0) / args.steps
    ms_per_step = elapsed_ms / args.steps
    counts[:] = [r[5] for r in recs]  # the candidate's valid blocks, as try_step reports them
    # kernel times at the end state: 10 back-to-back launches each between
    # two events (host launch work overlaps the previous launch's execution)
    lin_ms, solve_ms = [], []
    for fn, out in ((lambda: lv.linearize(lv.poses[lv.cur]), lin_ms),
                    (lambda: lv.solve(lv.cur, 1e-3, lv._status_solve_ptr), solve_ms)):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(10):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / 10)
    # e2e: host poses in, evaluate, the loop, poses + records out
    host_in = torch.from_numpy(snap_rows.copy()).pin_memory()
    gens_in = torch.from_numpy(snap_gens.copy()).pin_memory()
    rows_out = torch.empty_like(host_in).pin_memory()
    gens_out = torch.empty_like(gens_in).pin_memory()
    torch.cuda.synchronize()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    lv.cur = 0
    lv.poses[0].copy_(host_in, non_blocking=True)
    lv.gens[0].copy_(gens_in, non_blocking=True)
    c_, n_ = lv.evaluate_current()
    recs2, err2, _, _ = lv.lm_level_device(c_, n_, lam, _NoTermination, args.steps, float("inf"))
    rows_out.copy_(lv.poses[lv.cur], non_blocking=True)
    gens_out.copy_(lv.gens[lv.cur], non_blocking=True)
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / args.steps
    assert recs2 == [r[:4] for r in recs]  # the same iterations again
    rec_bytes = len(recs2) * 6 * 8 + 16 * 8
    e2e = {"value": total_pp / (e2e_ms / 1e3), "unit": "pixel-pairs/s",
           "h2d_bytes_per_step": int((host_in.numel() * 8 + gens_in.numel() * 4 + 16 * 8)
                                     / args.steps),
           "d2h_bytes_per_step": int((rows_out.numel() * 8 + gens_out.numel() * 4 + rec_bytes)
                                     / args.steps),
           "ms_per_step": e2e_ms,
           "path": "DeviceLevel.lm_level_device (one conditional-graph launch per level) via "
                   "the C ABI; poses in / out through pinned host buffers, once per call"}
    peak, peak_kind = measured_peak_hbm()
    lin_avg_ms = statistics.mean(lin_ms)
    achieved = total_pp * BYTES_PER_PIXEL_PAIR / (lin_avg_ms / 1e3) / 1e9
    trafficd = ncu_traffic(args.config)
    traffic = (trafficd["dram_bytes_per_pixel_pair"] * total_pp
               if trafficd and trafficd.get("dram_bytes_per_pixel_pair") else None)
    line = {
        "metric": METRIC,
        "value": total_pp / (ms_per_step / 1e3),
        "unit": "pixel-pairs/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(args.config, meta["cam"], meta["frames"], n_pairs, total_pp,
                                  solver),
        "parallelism": "single GPU, device-resident LM loop",
        "setup": {
            "l2": l2_note(store),
            "precision": "fp64 throughout (geometry, residuals, Jacobians, H/b/cost sums)",
            "gn_iteration_ms": ms_per_step,
            "setup_seconds": round(t_setup, 2),
            "graph_seconds": round(meta["graph_seconds"], 2),
            "initial_cost": cost0,
            "initial_valid_blocks": count0,
            "timed_loop": "one DeviceLevel.lm_level_device launch of --steps iterations "
                          "(conditional CUDA graph; accept/reject and lambda on the device)",
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
            "solve_ms": statistics.mean(solve_ms),
            "pcg_last_solve": None,
            "algorithmic_bytes_per_launch": total_pp * BYTES_PER_PIXEL_PAIR,
            "kernel_times": "10 back-to-back eager launches at the loop's end state",
        },
        "compute": compute_roofline(counts, lin_avg_ms),
        "e2e": e2e,
        "valid_blocks_per_s": statistics.mean(counts) / (ms_per_step / 1e3),
        "gpu_launches": int(round(launches)),
        "clocks": clocks.summary(),
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, args.frames, n_pairs, total_pp)
    if not args.no_e2e_api:
        cb = line.get("cpu_baseline") or {}
        line["e2e_api"] = e2e_api(args.config, args.frames, device, cb.get("linearize_rate"),
                                  cb.get("solve_seconds"))
    print(json.dumps(line), flush=True)
    return line


def e2e_api(name: str, frames: int | None, device, cpu_rate: float | None,
            cpu_solve_seconds: float | None):
    """The whole reference-facing call chain a user runs, from host rasters:
    build_pyramid(device=) over the (n, H, W) host intensity/depth arrays
    (H2D inside), build_graph(device=), then solve_hierarchical (3 levels,
    10 + 5 + 3 LM iterations at most) with the refined poses back on the
    host.  Inputs are rendered once beforehand (not timed).  Timed twice in
    the process: the first call includes the device allocations (cudaMalloc
    of ~25 GB), `seconds` is the second, which reuses them.  Beside it,
    the reference CPU path for the same solve extrapolated from the
    cpu_baseline's measured oracle rate (pixel-pairs/s per linearisation)
    plus a dense LU per LM iteration at each level."""
    import torch

    import paper_2303_16878_b200 as P
    from paper_2303_16878_b200 import scenes as S

    c = CONFIGS[name]
    n = frames or c["n"]
    scales = tuple(1.0 / f for f in c["factors"])
    sensors = []  # (cam, ext, host intensity, host depth, max_translation, sensor id)
    if c["kind"] == "room":
        gt = S.room_loop(n)
        specs = [(S.rgbd_160(), P.Pose.identity(), S.BoxScene(), c["max_translation"], "sensor0")]
    else:
        gt = S.corridor_trajectory(n, c["spacing"])
        scene = S.corridor_scene(c["spacing"] * n + 20.0)
        if c["kind"] == "tum":
            specs = [(S.tum_640(), P.Pose(FORWARD_CAMERA, [0.0, 0.0, 0.1]), scene,
                      c["max_translation"], "sensor0")]
        elif c["kind"] == "fused":
            specs = [(S.lidar_os0_128(), P.Pose(np.eye(3), [0.0, 0.0, -0.05]), scene,
                      c["max_translation"], "lidar0"),
                     (S.tum_640(), P.Pose(FORWARD_CAMERA, [0.1, 0.0, 0.1]), scene,
                      c["max_translation_rgbd"], "rgbd0")]
        else:
            cam = S.hdl64() if c["kind"] == "hdl64" else S.lidar_os0_128()
            ext = P.Pose.identity() if c["kind"] == "hdl64" else P.Pose(np.eye(3), [0.0, 0.0, -0.05])
            specs = [(cam, ext, scene, c["max_translation"], "sensor0")]
    guess = S.perturb(gt, 0.05, math.radians(2.0), 11)
    for cam, ext, scene, max_t, sid in specs:
        rows = S.sensor_rows(gt, ext).to(device)
        rays = S.unit_rays(cam, device)
        I, D = [], []
        for s0 in range(0, n, 64):
            inten, depth, _ = S.render_batch(scene, cam, rows[s0:s0 + 64], rays)
            I.append(inten.cpu())
            D.append(depth.cpu())
        sensors.append((cam, ext, torch.cat(I).numpy(), torch.cat(D).numpy(), max_t, sid))
        del rows, rays
    torch.cuda.synchronize(device)

    def run():
        problems = []
        for cam, ext, inten, depth, max_t, sid in sensors:
            pyrs = P.build_pyramids_device(inten, depth, cam, scales, device=device)
            nodes = [P.FrameNode(k, guess[k], pyrs[k], 0.1 * k, sid) for k in range(n)]
            sext = P.SensorExtrinsics(ext)
            g = P.build_graph(nodes, P.MatchCriteria(max_translation=max_t), extrinsics=sext,
                              device=device)
            problems.append(P.BAProblem(g, {sid: sext}))
        if len(problems) == 1:
            res = P.solve_hierarchical(problems[0])
        else:
            res = P.solve_fusion(problems[0], problems[1], P.COUPLED)
        return res, problems

    t0 = time.perf_counter()
    run()
    cold = time.perf_counter() - t0
    t0 = time.perf_counter()
    res, problems = run()
    warm = time.perf_counter() - t0
    out = {"seconds": warm, "seconds_first_call": cold, "lm_iterations": len(res.records),
           "iterations_per_level": res.iterations_per_level(),
           "final_error": res.final_error(),
           "h2d_bytes": int(sum(a.nbytes + b.nbytes for _, _, a, b, _, _ in sensors)),
           "d2h_bytes": int(n * 12 * 8),
           "path": "build_pyramid(device=) from host rasters + build_graph(device=) + "
                   "solve_hierarchical / solve_fusion(coupled); poses returned to the host"}
    if cpu_rate:
        # linearisations = one per LM iteration + the initial one per level
        per_level = {lv: problems_pixel_pairs(problems, lv) for lv in range(len(scales))}
        t_lu = cpu_solve_seconds or 0.0  # the measured LU of the same dimension 6(N-1)
        t = 0.0
        for lv, k in res.iterations_per_level().items():
            t += (k + 1) * per_level[lv] / cpu_rate + k * t_lu
        out["reference_seconds_extrapolated"] = t
        out["reference_basis"] = ("oracle C port rate of cpu_baseline x pixel-pairs of every "
                                  "linearisation of this solve + dense LU per iteration")
    return out


def valid_pixel_pairs_shard(problems, level, local_level):
    """Depth-valid source pixels of this rank's slice [pair_lo, pair_hi) of
    the concatenated edge list (problem 0's edges, then problem 1's: the
    DeviceLevel pair order, so fused c5 shards like the others)."""
    import paper_2303_16878_b200 as P

    lo, hi = local_level.pair_lo, local_level.pair_hi
    total, base = 0, 0
    for prob in problems:
        n = len(prob.graph.edges)
        a, b = max(lo - base, 0), min(hi - base, n)
        if b > a:
            g = P.MatchGraph(prob.graph.nodes, prob.graph.edges[a:b])
            total += valid_pixel_pairs(P.BAProblem(g, prob.extrinsics, prob.gauge_index), level)
        base += n
    return total


# ---------------------------------------------------------------------------
# reference arm: the oracle port on the host cores (rank 0 only)
# ---------------------------------------------------------------------------
def run_reference(args):
    """`--impl reference`: the reference path on the host cores (the oracle C
    port, since the reference itself is numpy and cannot run on the GPU box),
    on a host-built bounded sample (ReferenceSample) — no GPU, no product
    library.  ms_per_step is the measured wall time of each sample step;
    value is the full-iteration throughput extrapolated from it."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    world = int(os.environ.get("WORLD_SIZE", "1"))
    smp = ReferenceSample(args.config, args.frames)
    c = CONFIGS[args.config]
    if smp.full_pp is None:  # --frames override: no committed constants for that size
        raise SystemExit("--impl reference needs the configured frame count (or a whole sample)")
    for _ in range(args.warmup):
        smp.step()
    ts = [smp.step() for _ in range(args.steps)]
    walls = [t["wall"] for t in ts]
    its = [smp.iteration_seconds(t) for t in ts]
    it = statistics.median(its)
    v = smp.full_pp / it
    t_med = ts[its.index(sorted(its)[len(its) // 2])]
    solver = args.solver or c.get("solver", "cholesky")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": v,
        "unit": "pixel-pairs/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": statistics.mean(walls) * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(args.config, smp.cam, smp.n_full, smp.full_pairs, smp.full_pp,
                                  solver),
        "parallelism": f"host cores ({smp.threads} threads)",
        "gn_iteration_ms_extrapolated": it * 1e3,
        "sample_step_ms": {k: statistics.mean(t[k] for t in ts) * 1e3
                           for k in ("lin", "asm", "solve", "update", "wall")},
        "setup": {"setup_seconds": round(smp.setup_seconds, 2),
                  "inputs": "host-built: torch-CPU renders, numpy pyramids, host build_graph"},
        "cpu_baseline": {"value": v, "unit": "pixel-pairs/s", "cores": smp.threads,
                         "kind": "port", "sample": smp.describe(t_med)},
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
    ap.add_argument("--lm-loop", default="auto", choices=["auto", "host"],
                    help="auto: small single-GPU problems time the device-resident LM loop "
                         "(the path solve_hierarchical takes there); host: graph replays "
                         "driven from the host every step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e-api", action="store_true",
                    help="skip the full solve_hierarchical from host rasters")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
