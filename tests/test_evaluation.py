"""ATE evaluation (host-side) against the reference's
outputs on seeded trajectories (tests/golden/evaluation.npz) and the
behaviours of pkg/tests/test_evaluation.py:36-200."""

import numpy as np
import pytest

import paper_2303_16878_b200 as P
from paper_2303_16878_b200.evaluation import Trajectory
from tests.fixtures import GOLDEN


def _poses(rows):
    return [P.Pose.from_row(r) for r in rows]


def _random_rigid(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    return P.Pose.from_quat(rng.uniform(-2, 2, 3), q)


def _random_traj(rng, n=30):
    return Trajectory(np.cumsum(rng.uniform(0.05, 0.2, n)),
                      [_random_rigid(rng) for _ in range(n)])


@pytest.mark.parametrize("case", range(4))
def test_matches_reference(case):
    z = np.load(GOLDEN / "evaluation.npz")
    ref = Trajectory(z[f"ref_ts_{case}"], _poses(z[f"ref_{case}"]))
    est = Trajectory(z[f"est_ts_{case}"], _poses(z[f"est_{case}"]))
    assert P.associate(est, ref, 0.02) == [tuple(p) for p in z[f"pairs_{case}"].tolist()]
    rep = P.evaluate_ate(est, ref, 0.02)
    rmse, rot_rmse, matches = z[f"report_{case}"]
    assert rep.matches == matches
    assert abs(rep.rmse - rmse) <= 1e-12 * max(1.0, rmse)
    assert abs(rep.rotation_rmse - rot_rmse) <= 1e-9
    np.testing.assert_allclose(rep.alignment.as_row(), z[f"align_{case}"], atol=1e-12)
    assert P.ate_rmse(est, ref, 0.02) == rep.rmse


def test_associate_cases():
    rng = np.random.default_rng(61)
    t = _random_traj(rng)
    assert P.associate(t, t) == [(k, k) for k in range(len(t))]
    shifted = Trajectory(t.timestamps + 0.005, t.poses)
    assert P.associate(shifted, t, max_dt=0.02) == [(k, k) for k in range(len(t))]
    with pytest.raises(P.NoAssociationError):
        P.associate(Trajectory(t.timestamps + 1000.0, t.poses), t, max_dt=0.02)
    three = [P.Pose.identity()] * 3
    pairs = P.associate(Trajectory([0.0, 0.010, 0.5], three),
                        Trajectory([0.004, 0.496, 0.9], three), max_dt=0.02)
    assert pairs == [(0, 0), (2, 1)]


def test_horn_align_properties():
    rng = np.random.default_rng(65)
    pts = rng.uniform(-2, 2, (10, 3))
    g = P.horn_align(pts, pts)
    assert np.allclose(g.rotation, np.eye(3), atol=1e-12) and np.allclose(g.translation, 0, atol=1e-12)
    for _ in range(20):
        pts = rng.uniform(-2, 2, (8, 3))
        g = _random_rigid(rng)
        rec = P.horn_align(pts, pts @ g.rotation.T + g.translation)
        assert np.allclose(rec.rotation, g.rotation, atol=1e-10)
        assert np.allclose(rec.translation, g.translation, atol=1e-10)
    line = np.stack([np.linspace(0, 1, 5), np.zeros(5), np.zeros(5)], axis=-1)
    with pytest.raises(P.DegenerateAlignmentError):
        P.horn_align(line, line + 1.0)
    with pytest.raises(P.DegenerateAlignmentError):
        P.horn_align(line[:2], line[:2])
    with pytest.raises(ValueError):
        P.horn_align(pts[:, :2], pts[:, :2])
    # optimality against random candidates
    est = rng.uniform(-1, 1, (12, 3))
    ref = est @ _random_rigid(rng).rotation.T + rng.normal(0, 0.05, (12, 3))
    g = P.horn_align(est, ref)
    best = np.sum((ref - (est @ g.rotation.T + g.translation)) ** 2)
    for _ in range(100):
        c = _random_rigid(rng)
        assert best <= np.sum((ref - (est @ c.rotation.T + c.translation)) ** 2) + 1e-12


def test_ate_properties():
    rng = np.random.default_rng(68)
    t = _random_traj(rng)
    assert P.ate_rmse(t, t) < 1e-12
    for _ in range(5):
        g = _random_rigid(rng)
        moved = Trajectory(t.timestamps, [g.compose(p) for p in t.poses])
        assert P.ate_rmse(moved, t) < 1e-9
    noisy = Trajectory(t.timestamps.copy(),
                       [P.Pose(p.rotation, p.translation + rng.normal(0, 0.05, 3)) for p in t.poses])
    assert abs(P.ate_rmse(noisy, t) - P.ate_rmse(t, noisy)) < 1e-9
    rep = P.evaluate_ate(t, t)
    assert rep.rmse < 1e-12 and rep.rotation_rmse < 1e-6 and rep.matches == len(t)


def test_trajectory_validation():
    with pytest.raises(ValueError):
        Trajectory([0.0, 0.0], [P.Pose.identity()] * 2)
    with pytest.raises(ValueError):
        Trajectory([], [])
    with pytest.raises(ValueError):
        Trajectory([0.0, 1.0], [P.Pose.identity()])
