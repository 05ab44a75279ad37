"""cProfile of the c4 bench problem build (pyramids on the device + graph):
where the host time of the first build_graph call goes."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402

torch.zeros(1, device="cuda")
prof = cProfile.Profile()
prof.enable()
problems, guess, gt, meta = bench.build_problem("c4", torch.device("cuda", 0))
torch.cuda.synchronize()
prof.disable()
print("graph_seconds", meta["graph_seconds"])
st = pstats.Stats(prof)
st.sort_stats("cumulative").print_stats(35)
