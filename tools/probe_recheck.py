"""How many pixels K6 hands to the host eigh (normals recheck) per scan, and
what it costs: c4 OS0-128 scans and c3 640x480 frames."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_16878_b200 as P  # noqa: E402
from paper_2303_16878_b200 import pyramid_device as PD  # noqa: E402
from paper_2303_16878_b200 import scenes as S  # noqa: E402

dev = torch.device("cuda", 0)
for name, cam, ext, spacing in (("c4", S.lidar_os0_128(), P.Pose(np.eye(3), [0, 0, -0.05]), 2.0),
                                ("c3", S.tum_640(), P.Pose(bench.FORWARD_CAMERA, [0, 0, 0.1]), 0.05)):
    n = 64
    gt = S.corridor_trajectory(n, spacing)
    rows = S.sensor_rows(gt, ext).to(dev)
    _, depth, _ = S.render_batch(S.corridor_scene(spacing * n + 20), cam, rows)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.estimate_normals_device(depth, cam)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(name, "recheck pixels", PD.last_recheck_count, "of", depth.numel(),
          f"({PD.last_recheck_count / depth.numel():.2e}); {dt * 1e3:.1f} ms for {n} frames")
