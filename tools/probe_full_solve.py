"""Wall-clock of a full solve_hierarchical on a bench workload (device pyramids
and graph already built), with per-level iteration counts."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_16878_b200 as P  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c4"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 200
dev = torch.device("cuda", 0)
t0 = time.perf_counter()
problems, guess, gt, meta = bench.build_problem(cfg_name, dev, frames)
torch.cuda.synchronize()
t_setup = time.perf_counter() - t0
prob = problems[0]
for rep in range(2):
    t0 = time.perf_counter()
    res = P.solve_hierarchical(prob, P.SolverConfig(), initial=guess)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    levels = {}
    for r in res.records:
        levels.setdefault(r.level, 0)
        levels[r.level] += 1
    err = max(float(abs(p.translation - q.translation).max()) for p, q in zip(res.poses, gt))
    print(f"rep {rep}: solve_hierarchical {t:.2f} s, iterations per level {levels}, "
          f"level wall times {[(lv, round(s, 3)) for lv, s in res.level_times]}, "
          f"max |t - t_gt| {err:.2e} m (setup {t_setup:.1f} s)")
