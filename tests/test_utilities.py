"""The reference's public utilities beside the solver — `reproject`
(solver.py:154-176) and `sample` (cues.py:412-430) — against outputs of the
reference itself (tests/golden/utility.npz, tests/golden/make_golden.py
`utility`), and the drop-in surface: every name the reference exports."""
import numpy as np
import pytest

import paper_2303_16878_b200 as P
from tests import fixtures as F

# pkg/src/photoba/__init__.py:38-71 (the reference's __all__)
REFERENCE_ALL = [
    "BAProblem", "CueImage", "CuePyramid", "FrameNode", "Intrinsics", "MatchCriteria",
    "MatchGraph", "NormalConfig", "PerturbationVector", "PINHOLE", "Pose", "SensorExtrinsics",
    "SolveResult", "SolverConfig", "SPHERICAL", "Trajectory", "associate", "ate_rmse", "boxplus",
    "build_graph", "build_pyramid", "estimate_normals", "evaluate_ate", "exp", "horn_align",
    "overlap_ratio", "project", "projective_jacobian", "relative", "reproject", "sample", "skew",
    "solve_fusion", "solve_hierarchical", "solve_level", "unproject",
]


def test_every_reference_export_exists():
    missing = [n for n in REFERENCE_ALL if not hasattr(P, n)]
    assert not missing, missing
    assert set(REFERENCE_ALL) <= set(P.__all__)


@pytest.fixture(scope="module")
def gold():
    return F.load("utility")


@pytest.mark.parametrize("tag", ["pin", "sph"])
def test_reproject_matches_reference(gold, tag):
    cam = F.cam_from_row(gold[f"{tag}_cam"])
    xi, xj, off = (P.Pose.from_row(gold[f"{tag}_{k}"][0]) for k in ("xi", "xj", "off"))
    uv_dst, p_bar, valid = P.reproject(gold[f"{tag}_uv"], gold[f"{tag}_depth"], xi, xj,
                                       P.SensorExtrinsics(off), cam, cam)
    assert np.array_equal(valid, gold[f"{tag}_valid"])
    assert 0 < valid.sum() < valid.size or tag == "sph"
    np.testing.assert_allclose(p_bar, gold[f"{tag}_p_bar"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(uv_dst, gold[f"{tag}_uv_dst"], rtol=0, atol=1e-9)


def test_reproject_identity_is_a_round_trip():
    cam = P.Intrinsics(100.0, 95.0, 32.0, 24.0, 64, 48, P.PINHOLE, 0.1, 50.0)
    uv = np.array([[3.0, 4.0], [10.25, 30.5], [63.0, 47.0]])
    x = P.Pose(np.eye(3), [0.3, -0.2, 1.0])
    uv2, _, ok = P.reproject(uv, np.array([1.0, 2.0, 3.0]), x, x, P.SensorExtrinsics.identity(),
                             cam, cam)
    assert ok.all()
    np.testing.assert_allclose(uv2, uv, atol=1e-12)


@pytest.mark.parametrize("channel", ["intensity", "depth", "normals"])
def test_sample_matches_reference(gold, channel):
    cam = F.cam_from_row(gold["pin_cam"])
    img = P.CueImage(gold["img_I"], gold["img_D"], gold["img_N"], cam)
    uv = gold["sample_uv"]
    v, g, ok = P.sample(img, uv, channel)
    assert np.array_equal(ok, gold[f"sample_{channel}_ok"])
    assert 0 < ok.sum() < ok.size
    assert np.array_equal(v, gold[f"sample_{channel}_v"])
    assert np.array_equal(g, gold[f"sample_{channel}_g"])
    v1, g1, ok1 = P.sample(img, uv[5], channel)
    assert isinstance(ok1, bool) and ok1 == bool(gold[f"sample1_{channel}_ok"])
    assert np.array_equal(v1, gold[f"sample1_{channel}_v"])
    assert np.array_equal(g1, gold[f"sample1_{channel}_g"])


def test_sample_rejects_unknown_channel(gold):
    img = P.CueImage(gold["img_I"], gold["img_D"], gold["img_N"], F.cam_from_row(gold["pin_cam"]))
    with pytest.raises(ValueError):
        P.sample(img, np.zeros(2), "colour")
