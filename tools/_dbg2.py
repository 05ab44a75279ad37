import sys; sys.path.insert(0, '.')
import torch, bench, numpy as np
import paper_2303_16878_b200 as P
from paper_2303_16878_b200.device import DeviceLevel, FrameStore
cfgname = sys.argv[1]
dev = torch.device("cuda", 0)
problems, guess, _, meta = bench.build_problem(cfgname, dev)
lv = DeviceLevel(problems, meta["level"], P.SolverConfig(), FrameStore(dev))
rows, gens = P.se3.pose_rows(guess)
lv.set_poses(rows, gens)
class NoStop:
    lm_factor = 10.0
    termination_rel_decrease = -1.0
cost, count = lv.evaluate_current()
recs, err, _, _ = lv.lm_level_device(cost, count, 1e-3, NoStop, 30)
st = lv.lm_stamps.cpu().numpy().reshape(-1, 8)[1:len(recs) + 1]
d = np.diff(st[:, :6], axis=1) / 1e3
print(cfgname, "iterations", len(recs), "phase us (solve, apply, lin, asm, decide+copy):", np.round(np.median(d, axis=0), 1),
      "iteration total", np.round(np.median(np.diff(st[:, 0])) / 1e3, 1))
