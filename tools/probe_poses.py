"""Linearise timing at guess vs ground-truth poses (c4/200), back-to-back."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
import paper_2303_16878_b200 as P
from paper_2303_16878_b200.device import DeviceLevel, FrameStore

dev = torch.device("cuda", 0)
problems, guess, gt, meta = bench.build_problem("c4", dev, 200)
lv = DeviceLevel(problems, meta["level"], P.SolverConfig(), FrameStore(dev))
for name, poses in (("guess", guess), ("gt", gt), ("guess", guess)):
    rows, _ = P.se3.pose_rows(poses)
    pt = torch.from_numpy(rows).to(dev)
    recs = lv.linearize(pt)
    torch.cuda.synchronize()
    cnt = float(recs[:, 91].sum())
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        lv.linearize(pt)
    e1.record(); torch.cuda.synchronize()
    print(name, "valid blocks", int(cnt), "ms", round(e0.elapsed_time(e1) / 3, 3))
