"""Per-shard linearisation times of the multi-GPU split, measured on ONE GPU.

For world sizes 2/4/8 the c4 pair list is split exactly as
`distributed.make_level` splits it (`shard_ranges` over source-pixel
counts), and each rank's shard is linearised on its own, one after the
other, at the bench's operating point (the poses after the bench's warm-up
LM steps).  No shard waits on another, so this measures the work each GPU
would do, not a simulated collective.  The slowest shard bounds the
linearise part of an N-GPU iteration; the rank-0 solve, assembly and the
record gather / pose broadcast come on top (reported separately; the gather
is NOT measured here — one GPU).

    python tools/shard_projection.py [--config c4] [--reps 5]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_16878_b200 as P  # noqa: E402
from paper_2303_16878_b200 import distributed as D  # noqa: E402
from paper_2303_16878_b200.device import DeviceLevel, FrameStore  # noqa: E402


def time_linearize(level, poses, reps):
    out = []
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        level.linearize(poses)
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.mean(out[1:])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--frames", type=int, default=None)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup-steps", type=int, default=3)
    args = ap.parse_args()
    device = torch.device("cuda", 0)
    torch.cuda.set_device(device)
    problems, guess, gt, meta = bench.build_problem(args.config, device, args.frames)
    level = meta["level"]
    cfg = P.SolverConfig()
    store = FrameStore(device)
    full = DeviceLevel(problems, level, cfg, store)
    full.solve_events = []
    rows, gens = P.se3.pose_rows(guess)
    full.set_poses(rows, gens)
    cost, _ = full.evaluate_current()
    lam = cfg.lm_initial_lambda
    for _ in range(args.warmup_steps):  # the bench's warm-up: same operating point
        ok_s, ok_u, c, n = full.try_step(lam)
        if ok_s and ok_u and c < cost and n > 0:
            full.accept()
            cost, lam = c, max(lam * 0.5, 1e-12)
        else:
            lam *= cfg.lm_factor
    solve_ms = statistics.mean(a.elapsed_time(b) for a, b in full.solve_events)
    poses = full.poses[full.cur]
    one = time_linearize(full, poses, args.reps)
    px = D.pair_pixels(problems, level, cfg)
    result = {"config": args.config, "frames": meta["frames"], "pairs": len(px),
              "linearize_ms_1gpu": one, "solve_ms_rank0": solve_ms, "world": {}}
    for world in (2, 4, 8):
        ranges = D.shard_ranges(px, world)
        times = []
        for lo, hi in ranges:
            shard = DeviceLevel(problems, level, cfg, store, pair_range=(lo, hi), assemble=False)
            times.append(time_linearize(shard, poses, args.reps))
            del shard
        result["world"][world] = {
            "ranges": ranges, "shard_ms": times, "max_ms": max(times),
            "mean_ms": statistics.mean(times), "imbalance": max(times) / statistics.mean(times),
            "speedup_linearize": one / max(times),
            "projected_iteration_ms_excl_gather": max(times) + solve_ms,
        }
        print(world, [round(t, 2) for t in times], flush=True)
    print(json.dumps(result))
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/shard_projection.json", "w") as f:
        json.dump(result, f, indent=1)


if __name__ == "__main__":
    main()
