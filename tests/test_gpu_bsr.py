"""Block-sparse normal equations (pba_assemble_bsr, pba_solve_dense_bsr,
pba_solve_pcg_bsr) against the dense forms they replace: the same sums in
the same order (solver.py:428-449), so the blocks and the solves are
bit-identical."""
import math

import numpy as np
import pytest

import paper_2303_16878_b200 as P
from paper_2303_16878_b200 import native as N

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _level(gauge, solver="cholesky", n=10):
    from paper_2303_16878_b200 import scenes as S
    from paper_2303_16878_b200.device import DeviceLevel, FrameStore

    cam = S.rgbd_160()
    gt = S.room_loop(n)
    pyrs = S.host_pyramids(S.BoxScene(), cam, gt, P.Pose.identity(), (1.0,))
    guess = S.perturb(gt, 0.05, math.radians(2.0), 11)
    nodes = [P.FrameNode(k, guess[k], pyrs[k], 0.1 * k) for k in range(n)]
    prob = P.BAProblem(P.build_graph(nodes), gauge_index=gauge)
    lv = DeviceLevel([prob], 0, P.SolverConfig(linear_solver=solver),
                     FrameStore(torch.device("cuda", 0)))
    rows, gens = P.se3.pose_rows(guess)
    lv.set_poses(rows, gens)
    lv.evaluate_current()
    return lv


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _dense_assembly(lv):
    lib = N.load()
    dp, di, op, orc, oi = lv.plan
    H = torch.zeros((lv.dim, lv.dim), dtype=torch.float64, device="cuda")
    b = torch.zeros(lv.dim, dtype=torch.float64, device="cuda")
    tot = torch.zeros(2, dtype=torch.float64, device="cuda")
    N.check(lib.pba_assemble(lv.records.data_ptr(), lv.n_pairs_total, lv.n_free, dp.data_ptr(),
                             di.data_ptr(), lv.n_off, op.data_ptr(), orc.data_ptr(),
                             oi.data_ptr(), H.data_ptr(), b.data_ptr(), tot.data_ptr(),
                             _stream()), "assemble")
    return H, b, tot


@pytest.mark.parametrize("gauge", [0, 4, 9])
def test_bsr_assembly_equals_dense_assembly(gauge):
    lv = _level(gauge)
    H, b, tot = _dense_assembly(lv)
    Hd = lv.dense_H(lv.cur)
    assert torch.equal(Hd, H)
    assert torch.equal(lv.b[lv.cur], b)
    assert torch.equal(lv.totals[lv.cur], tot)
    # every stored block is a structurally non-zero block of H; nothing else is
    assert lv.n_blocks == lv.n_free + 2 * lv.n_off
    assert int((H.reshape(lv.n_free, 6, lv.n_free, 6).abs().sum((1, 3)) > 0).sum()) == lv.n_blocks


@pytest.mark.parametrize("solver", ["cholesky", "pcg"])
def test_bsr_solves_equal_dense_solves(solver):
    lib = N.load()
    lv = _level(3, solver)
    H, b, _ = _dense_assembly(lv)
    rp, cols, dblk, _ = lv.bsr
    lam = 1e-3
    d_bsr = torch.zeros(lv.dim, dtype=torch.float64, device="cuda")
    d_den = torch.zeros_like(d_bsr)
    st = torch.zeros(2, dtype=torch.int32, device="cuda")
    if solver == "cholesky":
        work = torch.empty(int(lib.pba_solve_work_bytes(lv.dim)), dtype=torch.uint8, device="cuda")
        N.check(lib.pba_solve_dense_bsr(lv.Hb[lv.cur].data_ptr(), rp.data_ptr(), cols.data_ptr(),
                                        b.data_ptr(), lv.dim, lam, None, lv.tile_env.ctypes.data,
                                        work.data_ptr(), 0, d_bsr.data_ptr(), st.data_ptr(),
                                        _stream()), "bsr")
        N.check(lib.pba_solve_dense(H.data_ptr(), b.data_ptr(), lv.dim, lam,
                                    lv.tile_env.ctypes.data, work.data_ptr(), d_den.data_ptr(),
                                    st[1:].data_ptr(), _stream()), "dense")
    else:
        work = torch.empty(int(lib.pba_pcg_work_bytes(lv.n_free)), dtype=torch.uint8,
                           device="cuda")
        info = torch.zeros(3, dtype=torch.float64, device="cuda")
        N.check(lib.pba_solve_pcg_bsr(lv.Hb[lv.cur].data_ptr(), b.data_ptr(), lv.n_free, lam,
                                      None, rp.data_ptr(), cols.data_ptr(), dblk.data_ptr(), 2000,
                                      1e-12, work.data_ptr(), d_bsr.data_ptr(), st.data_ptr(),
                                      info.data_ptr(), _stream()), "pcg bsr")
        N.check(lib.pba_solve_pcg(H.data_ptr(), b.data_ptr(), lv.n_free, lam, rp.data_ptr(),
                                  cols.data_ptr(), 2000, 1e-12, work.data_ptr(), d_den.data_ptr(),
                                  st[1:].data_ptr(), info.data_ptr(), _stream()), "pcg")
    torch.cuda.synchronize()
    assert st.tolist() == [0, 0]
    assert torch.equal(d_bsr, d_den)
    ref = np.linalg.solve(H.cpu().numpy() + lam * np.diag(np.diag(H.cpu().numpy())),
                          -b.cpu().numpy())
    assert np.max(np.abs(d_bsr.cpu().numpy() - ref)) <= 1e-8 * np.max(np.abs(ref))
