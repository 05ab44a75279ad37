#!/usr/bin/env python
"""Dataset loading throughput: load_dataset on the GPU (K7 decode + K6
pyramids) vs the host path (numpy, reference-exact), OS0-128 scans.

  python tools/dataset_bench.py [--frames 200] [--host-frames 4] [--dir /tmp/pba_ds]

Writes a synthetic dataset directory (rendered corridor scans, written with
the reference formats), then times both loaders end to end (file reads
included, page cache warm after the write).  Prints one JSON line.
"""

import argparse
import json
import shutil
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2303_16878_b200 as P  # noqa: E402
from paper_2303_16878_b200 import dataset as DS  # noqa: E402
from paper_2303_16878_b200 import scenes as S  # noqa: E402
from paper_2303_16878_b200.camera import SensorExtrinsics  # noqa: E402


def write(root: Path, n: int):
    cam = S.lidar_os0_128()
    poses = S.corridor_trajectory(n, 2.0)
    rows = S.sensor_rows(poses, P.Pose.identity()).cuda()
    frames = []
    for s0 in range(0, n, 64):
        inten, depth, _ = S.render_batch(S.corridor_scene(2.0 * n + 20.0), cam, rows[s0:s0 + 64])
        frames += [(inten[b].cpu().numpy(), depth[b].cpu().numpy()) for b in range(inten.shape[0])]
    m = DS.DatasetManifest([DS.SensorConfig("os0", cam, SensorExtrinsics.identity(), 0.001,
                                            "os0/intensity", "os0/depth")],
                           pyramid_scales=(0.25, 0.5, 1.0))
    tr = DS.Trajectory(np.arange(n) * 0.1, poses)
    DS.write_dataset(root, m, tr, {"os0": frames})
    return m, tr


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=200)
    ap.add_argument("--host-frames", type=int, default=4)
    ap.add_argument("--dir", default="/tmp/pba_ds")
    a = ap.parse_args()
    root = Path(a.dir)
    shutil.rmtree(root, ignore_errors=True)
    m, tr = write(root, a.frames)
    DS.load_dataset(root, device="cuda")  # warm-up (CUDA context, kernels)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    DS.load_dataset(root, device="cuda")
    torch.cuda.synchronize()
    dev_ms = (time.perf_counter() - t0) * 1e3 / a.frames
    # host path on a prefix (same files)
    small = root.parent / (root.name + "_host")
    shutil.rmtree(small, ignore_errors=True)
    small.mkdir()
    shutil.copy(root / "manifest", small / "manifest")
    sub = DS.Trajectory(tr.timestamps[:a.host_frames], tr.poses[:a.host_frames])
    DS.save_trajectory(sub, small / "trajectory.txt")
    for d in ("os0/intensity", "os0/depth"):
        (small / d).mkdir(parents=True)
        for ts in sub.timestamps:
            name = DS.timestamp_name(ts) + ".pgm"
            shutil.copy(root / d / name, small / d / name)
    t0 = time.perf_counter()
    DS.load_dataset(small)
    host_ms = (time.perf_counter() - t0) * 1e3 / a.host_frames
    print(json.dumps({"metric": "dataset_load_ms_per_scan", "frames": a.frames,
                      "device_ms_per_scan": round(dev_ms, 3), "host_ms_per_scan": round(host_ms, 1),
                      "speedup": round(host_ms / dev_ms, 1),
                      "bytes_per_scan": 2 * 2 * 128 * 1024,
                      "config": {"camera": "OS0-128 1024x128", "scales": [0.25, 0.5, 1.0],
                                 "note": "wall clock, file reads from a warm page cache"}}))
    shutil.rmtree(root, ignore_errors=True)
    shutil.rmtree(small, ignore_errors=True)


if __name__ == "__main__":
    main()
