"""Per-section cycle breakdown of the linearisation kernel (c4/200,
PBA_LIN_VARIANT=24 clock64 instrumentation), at guess and ground-truth poses."""
import ctypes
import os
import sys
from pathlib import Path

os.environ["PBA_LIN_VARIANT"] = "24"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_16878_b200 as P  # noqa: E402
from paper_2303_16878_b200 import native as N  # noqa: E402
from paper_2303_16878_b200.device import DeviceLevel, FrameStore  # noqa: E402

NAMES = ["src texel", "unproject+warp+project", "gather1+masks+occlusion",
         "normals+residuals+Huber", "Jacobian+I/D gradients", "accumulate (+N gradients)",
         "-", "rejected tail"]
dev = torch.device("cuda", 0)
problems, guess, gt, meta = bench.build_problem("c4", dev, 200)
lv = DeviceLevel(problems, meta["level"], P.SolverConfig(), FrameStore(dev))
lib = N.load()
cyc = (ctypes.c_uint64 * 8)()
cnt = (ctypes.c_uint64 * 8)()
for name, poses in (("guess", guess), ("gt", gt)):
    rows, _ = P.se3.pose_rows(poses)
    pt = torch.from_numpy(rows).to(dev)
    lv.linearize(pt)
    torch.cuda.synchronize()
    N.check(lib.pba_diag_section_cycles(cyc, cnt, 1), "diag")
    lv.linearize(pt)
    torch.cuda.synchronize()
    N.check(lib.pba_diag_section_cycles(cyc, cnt, 1), "diag")
    c = np.array(cyc[:], dtype=float)
    n = np.array(cnt[:], dtype=float)
    print(f"== {name}: total thread-cycles {c.sum():.3e}")
    for k in range(8):
        if n[k]:
            print(f"  {NAMES[k]:28s} visits {n[k]:.3e}  cycles/visit {c[k] / n[k]:8.1f}  share {c[k] / c.sum() * 100:5.1f}%")
