"""Time the one-CTA small solve (dim <= 64) on c1's level: block-sparse H
(pba_solve_dense_bsr) vs the same matrix dense (pba_solve_dense), warm,
back-to-back launches timed with CUDA events."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_16878_b200 as P  # noqa: E402
from paper_2303_16878_b200 import native as N  # noqa: E402
from paper_2303_16878_b200.device import DeviceLevel, FrameStore  # noqa: E402


def timed(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    dev = torch.device("cuda", 0)
    problems, guess, _, meta = bench.build_problem("c1", dev)
    lv = DeviceLevel(problems, meta["level"], P.SolverConfig(), FrameStore(dev))
    rows, gens = P.se3.pose_rows(guess)
    lv.set_poses(rows, gens)
    lv.evaluate_current()
    lib = N.load()
    st = torch.cuda.current_stream().cuda_stream
    rp, cols, _, _ = lv.bsr
    b = lv.b[lv.cur]
    H = lv.dense_H(lv.cur).contiguous()
    work = torch.empty(int(lib.pba_solve_work_bytes(lv.dim)), dtype=torch.uint8, device=dev)
    d = torch.zeros(lv.dim, dtype=torch.float64, device=dev)
    s = torch.zeros(1, dtype=torch.int32, device=dev)
    t_bsr = timed(lambda: lib.pba_solve_dense_bsr(lv.Hb[lv.cur].data_ptr(), rp.data_ptr(),
                                                  cols.data_ptr(), b.data_ptr(), lv.dim, 1e-3, None,
                                                  lv.tile_env.ctypes.data, work.data_ptr(), 0,
                                                  d.data_ptr(), s.data_ptr(), st))
    t_den = timed(lambda: lib.pba_solve_dense(H.data_ptr(), b.data_ptr(), lv.dim, 1e-3, None,
                                              work.data_ptr(), d.data_ptr(), s.data_ptr(), st))
    print(f"dim {lv.dim}: bsr {t_bsr:.1f} us, dense {t_den:.1f} us per call (back-to-back)")
    if hasattr(lib, "pba_hack_small_times"):  # an instrumented build (clock64 sections)
        import ctypes

        out = (ctypes.c_longlong * 8)()
        lib.pba_hack_small_times(out)
        print("cycles: stage", out[0], "factor", out[1], "substitute", out[2])



if __name__ == "__main__":
    main()
