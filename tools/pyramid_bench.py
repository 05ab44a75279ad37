#!/usr/bin/env python
"""Cue-pyramid build throughput: K6 on the GPU vs the host restatement.

  python tools/pyramid_bench.py [--frames 64] [--reps 5]

Renders OS0-128 corridor scans on the device, then times
build_pyramids_device (normals + three levels, factors 4/2/1) with CUDA
events, inputs resident in HBM; and the host build_pyramid (numpy, the
reference algorithm, bit-exact to it) on one scan.  Prints one JSON line.
"""

import argparse
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2303_16878_b200 as P  # noqa: E402
from paper_2303_16878_b200 import native as N  # noqa: E402
from paper_2303_16878_b200 import scenes as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    cam = S.lidar_os0_128()
    scales = (0.25, 0.5, 1.0)
    poses = S.corridor_trajectory(a.frames, 2.0)
    rows = S.sensor_rows(poses, P.Pose.identity()).cuda()
    inten, depth, _ = S.render_batch(S.corridor_scene(2.0 * a.frames + 20.0), cam, rows)
    P.build_pyramids_device(inten, depth, cam, scales)  # warm-up
    torch.cuda.synchronize()
    lib = N.load()
    l0 = lib.pba_kernel_launches()
    times = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        P.build_pyramids_device(inten, depth, cam, scales)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    launches = (lib.pba_kernel_launches() - l0) // a.reps
    times.sort()
    dev_ms = times[len(times) // 2] / a.frames
    hi, hd = inten[0].cpu().numpy(), depth[0].cpu().numpy()
    t0 = time.perf_counter()
    P.build_pyramid(hi, hd, cam, scales)
    host_ms = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"metric": "pyramid_build_ms_per_scan", "frames": a.frames,
                      "device_ms_per_scan": round(dev_ms, 4), "host_ms_per_scan": round(host_ms, 1),
                      "speedup": round(host_ms / dev_ms, 1), "launches_per_batch": int(launches),
                      "config": {"camera": "OS0-128 1024x128", "scales": scales}}))


if __name__ == "__main__":
    main()
