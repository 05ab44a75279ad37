"""Per-iteration time of an LM level on a small problem (c1 by default):
the bench's host-driven loop (step graph replay, synchronise, read the
scalars, decide on the host), the step graph replayed back to back with no
host work in between (a lower bound), and the device-resident loop
(DeviceLevel.lm_level_device: one conditional-graph launch runs all
iterations, decisions on the GPU)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_16878_b200 as P  # noqa: E402
from paper_2303_16878_b200.device import DeviceLevel, FrameStore  # noqa: E402


def main(config="c1", reps=200):
    dev = torch.device("cuda", 0)
    problems, guess, _, meta = bench.build_problem(config, dev)
    lv = DeviceLevel(problems, meta["level"], P.SolverConfig(), FrameStore(dev))
    rows, gens = P.se3.pose_rows(guess)
    lv.set_poses(rows, gens)
    lv.evaluate_current()
    lv.try_step(1e-3)
    lv.prepare_graphs()
    g = lv._graphs[lv.cur]
    for _ in range(10):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    dev_us = a.elapsed_time(b) / reps * 1e3
    t0 = time.perf_counter()
    for _ in range(reps):
        lv.try_step(1e-3)
    host_us = (time.perf_counter() - t0) / reps * 1e6
    # device-resident loop: `reps` iterations in one launch, no termination test
    class NoStop:
        lm_factor = 10.0
        termination_rel_decrease = -1.0

    cost, count = lv.evaluate_current()
    lv.lm_level_device(cost, count, 1e-3, NoStop, 5)  # capture + warm
    cost, count = lv.evaluate_current()
    torch.cuda.synchronize()
    a.record()
    recs, err, _, _ = lv.lm_level_device(cost, count, 1e-3, NoStop, reps)
    b.record()
    torch.cuda.synchronize()
    loop_us = a.elapsed_time(b) / max(len(recs), 1) * 1e3
    print(f"{config}: try_step loop {host_us:.1f} us/iteration; graph replay back to back "
          f"{dev_us:.1f}; device-resident loop {loop_us:.1f} ({len(recs)} iterations, error {err})")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["c1"]))
