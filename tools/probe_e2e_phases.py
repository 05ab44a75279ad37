"""Phases of the user-facing c4 call chain (bench.e2e_api's run(), warm):
device pyramids from host rasters, build_graph(device=), solve_hierarchical."""
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_16878_b200 as P  # noqa: E402
from paper_2303_16878_b200 import scenes as S  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    c = bench.CONFIGS["c4"]
    n = c["n"]
    scales = tuple(1.0 / f for f in c["factors"])
    gt = S.corridor_trajectory(n, c["spacing"])
    scene = S.corridor_scene(c["spacing"] * n + 20.0)
    cam = S.lidar_os0_128()
    ext = P.Pose(np.eye(3), [0.0, 0.0, -0.05])
    guess = S.perturb(gt, 0.05, math.radians(2.0), 11)
    rows = S.sensor_rows(gt, ext).to(dev)
    rays = S.unit_rays(cam, dev)
    inten, depth = [], []
    for s0 in range(0, n, 64):
        i_, d_, _ = S.render_batch(scene, cam, rows[s0:s0 + 64], rays)
        inten.append(i_.cpu())
        depth.append(d_.cpu())
    inten, depth = torch.cat(inten).numpy(), torch.cat(depth).numpy()
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pyrs = P.build_pyramids_device(inten, depth, cam, scales, device=dev)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        nodes = [P.FrameNode(k, guess[k], pyrs[k], 0.1 * k, "sensor0") for k in range(n)]
        sext = P.SensorExtrinsics(ext)
        g = P.build_graph(nodes, P.MatchCriteria(max_translation=c["max_translation"]),
                          extrinsics=sext, device=dev)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        if rep == 1 and "--profile" in sys.argv:
            import cProfile
            import pstats

            pr = cProfile.Profile()
            pr.enable()
        P.solve_hierarchical(P.BAProblem(g, {"sensor0": sext}))
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        if rep == 1 and "--profile" in sys.argv:
            pr.disable()
            pstats.Stats(pr).sort_stats("tottime").print_stats(25)
        print(f"rep {rep}: pyramids {t1 - t0:.3f} s, graph {t2 - t1:.3f} s, "
              f"solve {t3 - t2:.3f} s, total {t3 - t0:.3f} s")


if __name__ == "__main__":
    main()
