"""Does a full solve on a bench workload converge?  Prints the LM trace, pose
errors vs ground truth and the objective at the guess / final / ground-truth
poses.  (The oracle comparison at this sensor shape lives in
tests/test_gpu_parity.py::test_os0_128_full_resolution_records_and_trace_match_oracle.)"""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_16878_b200 as P  # noqa: E402

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
