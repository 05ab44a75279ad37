#!/usr/bin/env python
"""Small end-to-end workload for compute-sanitizer: every
kernel family of libpba_b200 on tiny inputs.

  compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_case.py

(one tool per gpurun call, tools/gpu_sanitize.sh).  Cases: c1 (10 x 160x120
pinhole, 24 pairs) through solve_hierarchical with the Cholesky solver and
with the cooperative block-Jacobi PCG; c4-shaped OS0-128 with 5 scans built
by the device pyramid builder (K6) and the device graph (K5), then LM steps
through the nested-dissection-free and the tiled solve; texel build (K0),
atan2 table and the dataset raster decode (K7)."""
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_16878_b200 as P  # noqa: E402
from paper_2303_16878_b200 import scenes as S  # noqa: E402


def c1_problem():
    cam = S.rgbd_160()
    gt = S.room_loop(10)
    pyrs = S.host_pyramids(S.BoxScene(), cam, gt, P.Pose.identity(), (0.5, 1.0))
    guess = S.perturb(gt, 0.05, math.radians(2.0), 11)
    nodes = [P.FrameNode(k, guess[k], pyrs[k], 0.1 * k) for k in range(10)]
    return P.BAProblem(P.build_graph(nodes), gauge_index=3)


def main():
    from paper_2303_16878_b200 import native as N

    print("checked library:", int(N.load().pba_build_checked()), flush=True)
    dev = torch.device("cuda", 0)
    prob = c1_problem()
    cfg = P.SolverConfig(max_iterations_per_level=(3, 3))
    r1 = P.solve_hierarchical(prob, cfg)
    r2 = P.solve_hierarchical(prob, P.SolverConfig(max_iterations_per_level=(3, 3),
                                                   linear_solver="pcg"))
    c, n = P.total_error(prob, r1.poses, 1)
    print("c1", len(r1.records), len(r2.records), c, n, flush=True)
    problems, guess, _, meta = bench.build_problem("c4", dev, 5)
    res = P.solve_level(problems[0], guess, meta["level"], max_iterations=2)
    print("c4/5", len(problems[0].graph.edges), [r.valid_blocks for r in res[1]], flush=True)
    from paper_2303_16878_b200 import native as N

    lib = N.load()
    y = torch.tensor([1.0, -1.0, 0.0, 3.0], dtype=torch.float64, device=dev)
    x = torch.tensor([0.5, 0.5, -1.0, 0.0], dtype=torch.float64, device=dev)
    out = torch.empty_like(y)
    N.check(lib.pba_atan2_batch(y.data_ptr(), x.data_ptr(), 4, out.data_ptr(),
                                torch.cuda.current_stream().cuda_stream), "atan2")
    raw = torch.from_numpy(np.arange(64, dtype=np.uint8)).to(dev)
    o = torch.empty(32, dtype=torch.float64, device=dev)
    N.check(lib.pba_decode_raster(raw.data_ptr(), 32, N.PBA_RASTER_U16_DEPTH, 0.001, o.data_ptr(),
                                  torch.cuda.current_stream().cuda_stream), "decode")
    # nested-dissection Cholesky on a banded system (the c4 solve's shape, smaller)
    dim, band = 2049, 20
    rng = np.random.default_rng(1)
    A = np.triu(np.tril(rng.normal(size=(dim, dim)), band), -band)
    H = A @ A.T + 1e-3 * np.eye(dim)
    T = (dim + 63) // 64
    first = np.array([(np.nonzero(H[r, : r + 1])[0][:1].tolist() or [r])[0] for r in range(dim)])
    env = np.array([first[t * 64: (t + 1) * 64].min() // 64 for t in range(T)], np.int32)
    Ht = torch.from_numpy(H).to(dev)
    bt = torch.from_numpy(rng.normal(size=dim)).to(dev)
    work = torch.empty(int(lib.pba_solve_work_bytes(dim)), dtype=torch.uint8, device=dev)
    delta = torch.zeros(dim, dtype=torch.float64, device=dev)
    st = torch.zeros(2, dtype=torch.int32, device=dev)
    N.check(lib.pba_solve_dense(Ht.data_ptr(), bt.data_ptr(), dim, 1e-3, env.ctypes.data,
                                work.data_ptr(), delta.data_ptr(), st.data_ptr(),
                                torch.cuda.current_stream().cuda_stream), "solve")
    torch.cuda.synchronize()
    assert int(st[0].item()) == 0
    print("sanitize case ok", flush=True)


if __name__ == "__main__":
    main()
