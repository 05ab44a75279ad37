"""The reference's behavioural solver tests (pkg/tests/test_solver.py:374-563)
run on the GPU path: same scenes (raw renders from the reference renderer in
tests/golden/behaviour.npz, pyramids rebuilt with the bit-exact host
build_pyramid), same seeded perturbations, same assertions."""
import math

import numpy as np
import pytest

import paper_2303_16878_b200 as P
from paper_2303_16878_b200.camera import Intrinsics
from paper_2303_16878_b200.evaluation import Trajectory
from tests.fixtures import GOLDEN

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

RGBD_EXT = P.SensorExtrinsics(P.Pose(np.eye(3), [0.0, 0.0, 0.1]))
LIDAR_EXT = P.SensorExtrinsics(P.Pose(np.eye(3), [0.0, 0.0, -0.05]))


@pytest.fixture(scope="module")
def z():
    return np.load(GOLDEN / "behaviour.npz")


def _cam(row):
    model = P.PINHOLE if row[6] == 0 else P.SPHERICAL
    return Intrinsics(row[0], row[1], row[2], row[3], int(row[4]), int(row[5]), model, row[7],
                      row[8])


def _pyr(z, tag, cam_key="cam_rgbd"):
    return P.build_pyramid(z[f"{tag}_I"], z[f"{tag}_D"], _cam(z[cam_key]), (0.125, 0.25, 0.5))


def _selfalign(pyr, gt, bad, sensor="sensor0", ext=None):
    nodes = [P.FrameNode(0, gt, pyr, 0.0, sensor), P.FrameNode(1, bad, pyr, 0.1, sensor)]
    exts = {sensor: ext} if ext is not None else {}
    return P.BAProblem(P.MatchGraph(nodes, [P.Edge(0, 1, P.COVISIBILITY)]), exts)


def _err(a, b):
    rel = P.relative(a, b)
    return float(np.linalg.norm(rel.translation)), P.rotation_angle(rel.rotation)


def test_zero_perturbation_terminates_immediately(z):
    I = P.Pose.identity()
    prob = _selfalign(_pyr(z, "zero"), I, I)
    poses, records = P.solve_level(prob, [I, I], 0)
    assert len(records) <= 2
    assert np.allclose(poses[1].matrix(), np.eye(4), atol=1e-9)


def test_two_frame_selfalign_recovers_pose(z):
    gt = P.Pose(np.eye(3), [-0.5, -0.3, -0.8])
    bad = P.Pose.from_row(z["selfalign_bad"][0])
    res = P.solve_hierarchical(_selfalign(_pyr(z, "selfalign"), gt, bad))
    et, er = _err(res.poses[1], gt)
    assert et < 1e-4 and er < 1e-4


def test_accepted_error_trace_is_monotone(z):
    gt = P.Pose(np.eye(3), [-0.5, -0.3, -0.8])
    bad = P.Pose.from_row(z["monotone_bad"][0])
    res = P.solve_hierarchical(_selfalign(_pyr(z, "selfalign"), gt, bad))
    for level in set(r.level for r in res.records):
        errors = [r.error for r in res.records if r.level == level]
        assert all(b <= a + 1e-15 for a, b in zip(errors, errors[1:]))


def test_already_optimal_hierarchical_is_identity_operation(z):
    gt = P.Pose(np.eye(3), [-0.4, 0.2, -0.5])
    res = P.solve_hierarchical(_selfalign(_pyr(z, "optimal"), gt, gt))
    assert np.allclose(res.poses[1].matrix(), gt.matrix(), atol=1e-9)


def test_small_recovery_improves_ate(z):
    gt_poses = [P.Pose.from_row(r) for r in z["loop_gt"]]
    guess = [P.Pose.from_row(r) for r in z["loop_guess"]]
    stamps = np.arange(5) * 0.1
    nodes = [P.FrameNode(k, guess[k], _pyr(z, f"loop{k}"), float(stamps[k])) for k in range(5)]
    res = P.solve_hierarchical(P.BAProblem(P.build_graph(nodes)))
    gt_t = Trajectory(stamps, gt_poses)
    assert P.ate_rmse(Trajectory(stamps, res.poses), gt_t) < 0.5 * P.ate_rmse(
        Trajectory(stamps, guess), gt_t)


def _fusion(z, gt, bad):
    prob_r = _selfalign(_pyr(z, "fusion_rgbd"), gt, bad, "rgbd", RGBD_EXT)
    prob_l = _selfalign(_pyr(z, "fusion_lidar", "cam_lidar"), gt, bad, "lidar", LIDAR_EXT)
    return prob_r, prob_l


def test_fusion_zero_perturbation_is_identity_both_modes(z):
    gt = P.Pose(np.eye(3), [-0.4, -0.2, -0.6])
    prob_r, prob_l = _fusion(z, gt, gt)
    for mode in (P.COUPLED, P.CONSECUTIVE):
        res = (P.solve_fusion(prob_r, prob_l, mode) if mode == P.COUPLED
               else P.solve_fusion(prob_l, prob_r, mode))
        et, er = _err(res.poses[1], gt)
        assert et < 1e-6 and er < 1e-6


def test_fusion_rejects_mismatched_lengths(z):
    gt = P.Pose(np.eye(3), [-0.4, -0.2, -0.6])
    prob_r, prob_l = _fusion(z, gt, gt)
    prob_l.graph.nodes.append(prob_l.graph.nodes[1])
    with pytest.raises(P.FusionConfigError):
        P.solve_fusion(prob_r, prob_l, P.COUPLED)


def test_coupled_converges_where_pinhole_fails(z):
    gt = P.Pose(np.eye(3), [-0.4, -0.2, -0.6])
    bad = P.Pose.from_row(z["coupled_bad"][0])
    prob_r, prob_l = _fusion(z, gt, bad)
    res_pin = P.solve_hierarchical(prob_r)
    res_cpl = P.solve_fusion(prob_r, prob_l, P.COUPLED)
    et, er = _err(res_pin.poses[1], gt)
    assert not (et < 1e-3 and er < 1e-3)
    et, er = _err(res_cpl.poses[1], gt)
    assert et < 1e-3 and er < 1e-3
    assert math.isfinite(res_cpl.records[-1].error)


# ---------------------------------------------------------------------------
# CUDA-graph LM step (device.DeviceLevel.try_step): identical to eager steps
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("solver", ["cholesky", "pcg"])
def test_graph_replayed_steps_equal_eager_steps(monkeypatch, solver):
    import math

    import torch

    from paper_2303_16878_b200 import scenes as S
    from paper_2303_16878_b200.device import DeviceLevel, FrameStore

    cam = S.rgbd_160()
    gt = S.room_loop(10)
    pyrs = S.host_pyramids(S.BoxScene(), cam, gt, P.Pose.identity(), (1.0,))
    guess = S.perturb(gt, 0.05, math.radians(2.0), 11)
    nodes = [P.FrameNode(k, guess[k], pyrs[k], 0.1 * k) for k in range(10)]
    prob = P.BAProblem(P.build_graph(nodes), gauge_index=2)
    cfg = P.SolverConfig(linear_solver=solver)
    rows, gens = P.se3.pose_rows(guess)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("PBA_GRAPH", mode)
        lv = DeviceLevel([prob], 0, cfg, FrameStore(torch.device("cuda", 0)))
        lv.set_poses(rows, gens)
        cost, _ = lv.evaluate_current()
        lam, trace = 1e-3, []
        for _ in range(8):  # accepted and rejected steps, so both buffers are used
            ok_s, ok_u, c, n = lv.try_step(lam)
            trace.append((ok_s, ok_u, c, n))
            if ok_s and ok_u and c < cost and n > 0:
                lv.accept()
                cost, lam = c, max(lam * 0.5, 1e-12)
            else:
                lam *= 10.0
        out[mode] = (trace, lv.current_rows()[0], lv.graph_launches_replayed)
    assert out["0"][0] == out["1"][0]
    assert np.array_equal(out["0"][1], out["1"][1])
    assert out["0"][2] == 0
    if solver == "cholesky":
        assert out["1"][2] > 0  # the replayed path really ran


# ---------------------------------------------------------------------------
# Device-resident LM level (csrc/lmloop.cu): one conditional-graph launch per
# level, identical to the host-driven loop
# ---------------------------------------------------------------------------
def _room_level_problem(gauge, n=10, scales=(1.0,)):
    import math

    from paper_2303_16878_b200 import scenes as S

    cam = S.rgbd_160()
    gt = S.room_loop(n)
    pyrs = S.host_pyramids(S.BoxScene(), cam, gt, P.Pose.identity(), scales)
    guess = S.perturb(gt, 0.05, math.radians(2.0), 11)
    nodes = [P.FrameNode(k, guess[k], pyrs[k], 0.1 * k) for k in range(n)]
    return P.BAProblem(P.build_graph(nodes), gauge_index=gauge), guess


@pytest.mark.parametrize("gauge,max_it", [(0, 10), (4, 10), (2, 3), (2, 1)])
def test_device_lm_loop_equals_host_loop(monkeypatch, gauge, max_it):
    import torch

    from paper_2303_16878_b200.bundle import _lm_level, _Runtime

    prob, guess = _room_level_problem(gauge)
    rows, gens = P.se3.pose_rows(guess)
    cfg = P.SolverConfig()
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("PBA_LM_DEVICE", mode)
        backend = _Runtime().level([prob], 0, cfg)
        backend.set_poses(rows, gens)
        recs = _lm_level(backend, 0, cfg, max_it)
        out[mode] = (recs, backend.current_rows(), backend.lm_device_iterations)
        del backend
        torch.cuda.synchronize()
    assert out["0"][2] == 0 and out["1"][2] == len(out["1"][0]) > 0  # the loop ran on the GPU
    assert out["1"][0] == out["0"][0]  # every IterationRecord field equal
    assert any(not r.accepted for r in out["1"][0]) or max_it < 10
    assert np.array_equal(out["1"][1][0], out["0"][1][0])
    assert np.array_equal(out["1"][1][1], out["0"][1][1])


def test_device_lm_loop_whole_solve_equals_host_loop(monkeypatch):
    prob, _ = _room_level_problem(3, scales=(0.5, 1.0))
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("PBA_LM_DEVICE", mode)
        res[mode] = P.solve_hierarchical(prob, P.SolverConfig())
    assert res["1"].records == res["0"].records
    assert all(np.array_equal(a.as_row(), b.as_row())
               for a, b in zip(res["1"].poses, res["0"].poses))


def test_device_lm_loop_with_pcg_matches_host_loop(monkeypatch):
    """The PCG solve's cooperative launch may not be capturable into the loop
    body; either way the level's records equal the host-driven loop's."""
    import torch

    from paper_2303_16878_b200.bundle import _lm_level, _Runtime

    prob, guess = _room_level_problem(1)
    rows, gens = P.se3.pose_rows(guess)
    cfg = P.SolverConfig(linear_solver="pcg")
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("PBA_LM_DEVICE", mode)
        backend = _Runtime().level([prob], 0, cfg)
        backend.set_poses(rows, gens)
        out[mode] = (_lm_level(backend, 0, cfg, 6), backend.current_rows()[0])
        del backend
        torch.cuda.synchronize()
    assert out["1"][0] == out["0"][0]
    assert np.array_equal(out["1"][1], out["0"][1])


def _decide_once(cost, count, lam, iteration, max_iterations, status_solve, status_step,
                 new_cost, new_count, rel_tol=1e-4):
    """One pba_lm_decide run as the whole body of a conditional loop graph."""
    import ctypes

    import torch

    from paper_2303_16878_b200 import native as N

    lib = N.load()
    dev = torch.device("cuda", 0)
    st = torch.zeros(N.LM_STATE_DOUBLES, dtype=torch.float64)
    st[N.LM_COST], st[N.LM_COUNT], st[N.LM_LAMBDA] = cost, count, lam
    st[N.LM_FACTOR], st[N.LM_REL_TOL] = 10.0, rel_tol
    st[N.LM_LAMBDA_CEILING], st[N.LM_COST_FLOOR] = 1e12, 1e-18
    st[N.LM_ITERATION], st[N.LM_MAX_ITERATIONS] = iteration, max_iterations
    state = st.to(dev)
    records = torch.zeros(N.LM_RECORD_DOUBLES * 8, dtype=torch.float64, device=dev)
    s_solve = torch.tensor([status_solve], dtype=torch.int32, device=dev)
    s_step = torch.tensor([status_step], dtype=torch.int32, device=dev)
    totals = torch.tensor([new_cost, new_count], dtype=torch.float64, device=dev)
    lam_dev = torch.zeros(1, dtype=torch.float64, device=dev)
    src = torch.arange(1.0, 7.0, dtype=torch.float64, device=dev)
    dst = torch.zeros(6, dtype=torch.float64, device=dev)
    d_arr = (ctypes.c_void_p * 1)(dst.data_ptr())
    s_arr = (ctypes.c_void_p * 1)(src.data_ptr())
    n_arr = (ctypes.c_int64 * 1)(48)
    stream = torch.cuda.Stream(dev)
    torch.cuda.synchronize()
    loop, handle = ctypes.c_void_p(), ctypes.c_uint64()
    N.check(lib.pba_lm_loop_begin(stream.cuda_stream, ctypes.byref(loop), ctypes.byref(handle)),
            "begin")
    N.check(lib.pba_lm_decide(state.data_ptr(), records.data_ptr(), s_solve.data_ptr(),
                              s_step.data_ptr(), totals.data_ptr(), lam_dev.data_ptr(),
                              handle.value, d_arr, s_arr, n_arr, 1, stream.cuda_stream), "decide")
    N.check(lib.pba_lm_loop_end(loop), "end")
    N.check(lib.pba_lm_loop_launch(loop, stream.cuda_stream), "launch")
    stream.synchronize()
    lib.pba_lm_loop_destroy(loop)
    out = state.cpu().numpy()
    n = int(out[N.LM_N_RECORDS])
    return out, records.cpu().numpy().reshape(-1, N.LM_RECORD_DOUBLES)[:n], float(lam_dev.item()), \
        dst.cpu().numpy()


def test_lm_decide_kernel_branches():
    """lm_decide_kernel against bundle._lm_level's branches (solver.py:505-537):
    singular first solve, singular later solve, ||dq|| >= 1, accept, reject,
    relative-decrease stop, iteration cap; the candidate is copied only on
    acceptance."""
    from paper_2303_16878_b200 import native as N

    # singular first solve -> UnderConstrainedError, no record
    s, r, _, dst = _decide_once(10.0, 3, 1e-3, 1, 10, 1, 0, 0.0, 0)
    assert s[N.LM_ERROR] == N.LM_ERR_UNDERCONSTRAINED and s[N.LM_STOP] == 1 and len(r) == 0
    # singular later solve -> lambda x factor, record, continue (cap stops this one)
    s, r, lam, dst = _decide_once(10.0, 3, 1e-3, 4, 4, 1, 0, 0.0, 0)
    assert s[N.LM_ERROR] == 0 and lam == 1e-3 * 10.0
    assert r.tolist() == [[1e-3 * 10.0, 10.0, 3.0, 0.0, 0.0, 0.0]] and not dst.any()
    # ||dq|| >= 1 -> InvalidPerturbationError
    s, r, _, _ = _decide_once(10.0, 3, 1e-3, 2, 10, 0, 1, 5.0, 3)
    assert s[N.LM_ERROR] == N.LM_ERR_PERTURBATION and s[N.LM_STOP] == 1 and len(r) == 0
    # accepted: cost / count move, lambda halves, candidate copied; cap stops
    s, r, lam, dst = _decide_once(10.0, 3, 1e-3, 1, 1, 0, 0, 5.0, 4)
    assert s[N.LM_ACCEPTED] == 1 and lam == max(1e-3 * 0.5, 1e-12)
    assert r.tolist() == [[lam, 5.0, 4.0, 1.0, 5.0, 4.0]]
    assert (s[N.LM_COST], s[N.LM_COUNT]) == (5.0, 4.0) and dst.tolist() == [1, 2, 3, 4, 5, 6]
    # rejected (no decrease, or count 0): lambda x factor, nothing copied
    for new_cost, new_count in ((20.0, 3), (5.0, 0)):
        s, r, lam, dst = _decide_once(10.0, 3, 1e-3, 1, 1, 0, 0, new_cost, new_count)
        assert s[N.LM_ACCEPTED] == 0 and lam == 1e-3 * 10.0 and not dst.any()
        assert (s[N.LM_COST], s[N.LM_COUNT]) == (10.0, 3.0)
    # relative decrease below the tolerance stops after accepting
    s, r, _, _ = _decide_once(10.0, 3, 1e-3, 1, 10, 0, 0, 10.0 * (1 - 1e-6), 3)
    assert s[N.LM_ACCEPTED] == 1 and s[N.LM_STOP] == 1 and s[N.LM_ITERATION] == 2
    # lambda above the ceiling stops after rejecting
    s, r, lam, _ = _decide_once(10.0, 3, 2e11, 1, 10, 0, 0, 20.0, 3)
    assert lam == 2e12 and s[N.LM_STOP] == 1
