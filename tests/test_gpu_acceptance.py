"""The reference's acceptance criteria (pkg/tests/test_acceptance.py:60-255)
on the GPU path, with the reference's own inputs (tests/golden/
acceptance.npz: raw renders and seeded perturbations; pyramids rebuilt with
the bit-exact host build_pyramid): synthetic recovery, iteration-count
sanity, hierarchical benefit, fusion ordering."""
import math

import numpy as np
import pytest

import paper_2303_16878_b200 as P
from paper_2303_16878_b200.camera import Intrinsics
from paper_2303_16878_b200.evaluation import Trajectory
from tests.fixtures import GOLDEN

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

RGBD = Intrinsics(55.0, 55.0, 64.0, 48.0, 128, 96, P.PINHOLE, 0.1, 50.0)  # rigs.rgbd_cam
RGBD_EXT = P.SensorExtrinsics(P.Pose(np.eye(3), [0.0, 0.0, 0.1]))
LIDAR_EXT = P.SensorExtrinsics(P.Pose(np.eye(3), [0.0, 0.0, -0.05]))


@pytest.fixture(scope="module")
def z():
    return np.load(GOLDEN / "acceptance.npz")


def _poses(rows):
    return [P.Pose.from_row(r) for r in rows]


@pytest.fixture(scope="module")
def recovery(z):
    gt = _poses(z["loop10_gt"])
    stamps = z["loop10_stamps"]
    guess = _poses(z["loop10_guess"])
    pyrs = [P.build_pyramid(z[f"loop10_{k}_I"], z[f"loop10_{k}_D"], RGBD) for k in range(10)]
    nodes = [P.FrameNode(k, guess[k], pyrs[k], float(stamps[k])) for k in range(10)]
    result = P.solve_hierarchical(P.BAProblem(P.build_graph(nodes)), P.SolverConfig())
    gt_t = Trajectory(stamps, gt)
    return {"result": result, "initial_ate": P.ate_rmse(Trajectory(stamps, guess), gt_t),
            "final_ate": P.ate_rmse(Trajectory(stamps, result.poses), gt_t)}


def test_synthetic_recovery_ninety_percent(recovery):
    assert recovery["final_ate"] <= 0.10 * recovery["initial_ate"]
    records = recovery["result"].records
    for level in sorted(set(r.level for r in records)):
        errors = [r.error for r in records if r.level == level]
        assert all(b <= a + 1e-15 for a, b in zip(errors, errors[1:]))


def test_iteration_counts_in_band(recovery):
    result = recovery["result"]
    counts = result.iterations_per_level()
    assert 3 <= counts.get(result.level_indices[0], 0) <= 20
    assert 1 <= counts.get(result.level_indices[-1], 0) <= 6


def test_three_level_schedule_beats_finest_only(z):
    gt = _poses(z["loop10_gt"])[:3]
    stamps = z["loop10_stamps"][:3]
    pyrs = [P.build_pyramid(z[f"loop10_{k}_I"], z[f"loop10_{k}_D"], RGBD) for k in range(3)]
    guess = list(gt)
    guess[2] = P.Pose.from_row(z["benefit_bad2"][0])
    gt_t = Trajectory(stamps, gt)
    initial = P.ate_rmse(Trajectory(stamps, guess), gt_t)
    nodes = [P.FrameNode(k, guess[k], pyrs[k], float(stamps[k])) for k in range(3)]
    problem = P.BAProblem(P.build_graph(nodes))
    full = P.solve_hierarchical(problem, P.SolverConfig())
    fine = P.solve_hierarchical(problem, P.SolverConfig(max_iterations_per_level=(30,)),
                                levels=[2])
    assert P.ate_rmse(Trajectory(stamps, full.poses), gt_t) < 0.20 * initial
    assert P.ate_rmse(Trajectory(stamps, fine.poses), gt_t) > 0.50 * initial


def test_fusion_basin_superset_and_consecutive_error():
    b = np.load(GOLDEN / "behaviour.npz")
    lidar_row = b["cam_lidar"]
    lidar = Intrinsics(lidar_row[0], lidar_row[1], lidar_row[2], lidar_row[3], int(lidar_row[4]),
                       int(lidar_row[5]), P.SPHERICAL, lidar_row[7], lidar_row[8])
    pyr_r = P.build_pyramid(b["fusion_rgbd_I"], b["fusion_rgbd_D"], RGBD)
    pyr_l = P.build_pyramid(b["fusion_lidar_I"], b["fusion_lidar_D"], lidar)
    gt = P.Pose(np.eye(3), [-0.4, -0.2, -0.6])
    bads = _poses(np.load(GOLDEN / "acceptance.npz")["fusion_grid_bad"])
    cfg = P.SolverConfig()
    modes = ("pinhole", "spherical", "coupled", "consecutive")
    errors = {m: np.zeros((25, 2)) for m in modes}

    def selfalign(pyr, bad, sensor, ext):
        nodes = [P.FrameNode(0, gt, pyr, 0.0, sensor), P.FrameNode(1, bad, pyr, 0.1, sensor)]
        return P.BAProblem(P.MatchGraph(nodes, [P.Edge(0, 1, P.COVISIBILITY)]), {sensor: ext})

    for c, bad in enumerate(bads):
        prob_r = selfalign(pyr_r, bad, "rgbd", RGBD_EXT)
        prob_l = selfalign(pyr_l, bad, "lidar", LIDAR_EXT)
        for mode in modes:
            if mode == "pinhole":
                res = P.solve_hierarchical(prob_r, cfg)
            elif mode == "spherical":
                res = P.solve_hierarchical(prob_l, cfg)
            elif mode == "coupled":
                res = P.solve_fusion(prob_r, prob_l, P.COUPLED, cfg)
            else:
                res = P.solve_fusion(prob_l, prob_r, P.CONSECUTIVE, cfg)
            err = P.relative(res.poses[1], gt)
            errors[mode][c] = (np.linalg.norm(err.translation),
                               abs(math.acos(np.clip((np.trace(err.rotation) - 1) / 2, -1, 1))))
    conv = {m: (errors[m][:, 0] <= 1e-3) & (errors[m][:, 1] <= 1e-3) for m in modes}
    assert (conv["coupled"] | ~conv["pinhole"]).all()
    all_ok = conv["pinhole"] & conv["spherical"] & conv["coupled"] & conv["consecutive"]
    assert all_ok.any()
    floor = 1e-6
    geo = {m: np.sqrt(errors[m][:, 0] * errors[m][:, 1]) for m in modes}
    cons = np.maximum(geo["consecutive"], floor)
    best = np.maximum(np.minimum(geo["pinhole"], geo["spherical"]), floor)
    assert (cons[all_ok] <= 1.05 * best[all_ok]).all()
