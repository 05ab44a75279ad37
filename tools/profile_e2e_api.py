"""cProfile of bench.e2e_api on c4 (host-side hotspots of the user-facing
call chain: pyramids from host rasters, device graph, solve_hierarchical)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
bench.e2e_api("c4", None, dev, None, None)  # warm (first call allocates)
pr = cProfile.Profile()
pr.enable()
out = bench.e2e_api("c4", None, dev, None, None)
pr.disable()
print("seconds", out["seconds"], "first", out["seconds_first_call"])
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
st = pstats.Stats(pr)
st.print_callers("method 'cpu'")
st.print_callers("__init__\\)$")
