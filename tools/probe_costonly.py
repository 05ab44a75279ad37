"""Time pba_linearize with and without Jacobians on the c4 bench problem."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch, numpy as np
import bench
import paper_2303_16878_b200 as P
from paper_2303_16878_b200.device import DeviceLevel, FrameStore

dev = torch.device("cuda", 0)
problems, guess, gt, meta = bench.build_problem("c4", dev, int(sys.argv[1]) if len(sys.argv) > 1 else 200)
lv = DeviceLevel(problems, meta["level"], P.SolverConfig(), FrameStore(dev))
rows, _ = P.se3.pose_rows(guess)
pt = torch.from_numpy(rows).to(dev)
for want in (True, False, True, False):
    lv.linearize(pt, want)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        lv.linearize(pt, want)
    e1.record(); torch.cuda.synchronize()
    print("want_jacobians", want, "ms", e0.elapsed_time(e1) / 3)
