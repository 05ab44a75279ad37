"""Does a full solve on a bench workload converge?  Prints the LM trace, pose
errors vs ground truth, the objective at the guess / final / ground-truth
poses, and checks a few pairs' GPU records against the oracle."""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_16878_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2303_16878_b200.device import DeviceLevel, FrameStore  # noqa: E402
from tests import fixtures as F  # noqa: E402

dev = torch.device("cuda", 0)
problems, guess, gt, meta = bench.build_problem(sys.argv[1] if len(sys.argv) > 1 else "c4", dev,
                                                int(sys.argv[2]) if len(sys.argv) > 2 else 200,
                                                normals=sys.argv[3] if len(sys.argv) > 3 else "estimate")
prob = problems[0]
res = P.solve_hierarchical(prob, P.SolverConfig(), initial=guess)
for r in res.records:
    print(r.format_line())
ef = np.array([np.abs(p.translation - q.translation).max() for p, q in zip(res.poses, gt)])
print("final pose err max/median", ef.max(), np.median(ef))
L = len(prob.graph.nodes[0].pyramid.levels)
for l in range(L):
    print("level", l, "cost guess/final/gt",
          [P.total_error(prob, poses, l) for poses in (guess, res.poses, gt)])
# a few pairs against the oracle at the final poses, finest level
sub = P.BAProblem(P.MatchGraph(prob.graph.nodes, prob.graph.edges[:6]), prob.extrinsics)
rows, _ = P.se3.pose_rows(res.poses)
got = DeviceLevel([sub], L - 1, P.SolverConfig(), FrameStore(dev)).linearize(
    torch.from_numpy(rows).to(dev)).cpu().numpy()
ref = O.OracleLevel([sub], L - 1, P.SolverConfig()).records(rows)
F.compare_records(got, ref)
print("6 pairs at full resolution match the oracle")
