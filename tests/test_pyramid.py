"""Host cue-pyramid builder: estimate_normals and
build_pyramid against the reference's own outputs (tests/golden/pyramid.npz,
made by tests/golden/make_golden.py) and the behaviours pinned by the
reference tests (pkg/tests/test_cues.py:45-195)."""

import math

import numpy as np
import pytest

import paper_2303_16878_b200 as P
from paper_2303_16878_b200.camera import Intrinsics

from tests.fixtures import GOLDEN


def _cam(row):
    model = P.PINHOLE if row[6] == 0 else P.SPHERICAL
    return Intrinsics(row[0], row[1], row[2], row[3], int(row[4]), int(row[5]), model, row[7],
                      row[8])


def _pinhole(w=64, h=48, f=60.0):
    return Intrinsics(f, f, w / 2.0, h / 2.0, w, h, P.PINHOLE, 0.1, 50.0)


def _spherical(w=128, h=32):
    return Intrinsics(w / (2 * math.pi), h / (math.pi / 2), w / 2.0, h / 2.0, w, h, P.SPHERICAL,
                      0.2, 80.0)


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN / "pyramid.npz")


@pytest.mark.parametrize("tag", ["p", "s"])
def test_normals_match_reference_bit_exact(golden, tag):
    cam = _cam(golden[f"{tag}_cam"])
    n = P.estimate_normals(golden[f"{tag}_D"], cam)
    ref = golden[f"{tag}_normals"]
    assert (np.linalg.norm(ref, axis=-1) > 0.5).sum() > 1000
    np.testing.assert_array_equal(n, ref)


@pytest.mark.parametrize("tag", ["p", "s"])
def test_pyramid_matches_reference_bit_exact(golden, tag):
    cam = _cam(golden[f"{tag}_cam"])
    scales = tuple(golden[f"{tag}_scales"])
    pyr = P.build_pyramid(golden[f"{tag}_I"], golden[f"{tag}_D"], cam, scales)
    assert pyr.scales == scales
    for l, img in enumerate(pyr.levels):
        np.testing.assert_array_equal(img.intensity, golden[f"{tag}_I_{l}"])
        np.testing.assert_array_equal(img.depth, golden[f"{tag}_D_{l}"])
        np.testing.assert_array_equal(img.normals, golden[f"{tag}_N_{l}"])
        k = img.intrinsics
        np.testing.assert_array_equal(
            [k.fx, k.fy, k.cx, k.cy, k.width, k.height, k.depth_min, k.depth_max],
            golden[f"{tag}_cam_{l}"][[0, 1, 2, 3, 4, 5, 7, 8]])


def test_plane_normals_point_at_camera():
    cam = _pinhole()
    n = P.estimate_normals(np.full((48, 64), 2.0), cam)
    ok = np.linalg.norm(n, axis=-1) > 0.5
    assert ok.mean() > 0.9
    assert np.abs(n[ok] - [0.0, 0.0, -1.0]).max() < 1e-3


def test_isolated_return_gets_no_normal():
    depth = np.zeros((48, 64))
    depth[20, 30] = 2.0
    assert not P.estimate_normals(depth, _pinhole()).any()


def test_no_valid_depth_gives_zero_field():
    depth = np.full((48, 64), np.nan)
    n = P.estimate_normals(depth, _pinhole())
    assert n.shape == (48, 64, 3) and not n.any()


def test_sphere_from_center_normals_are_radial():
    cam = _spherical()
    depth = np.full((32, 128), 5.0)
    n = P.estimate_normals(depth, cam)
    ok = np.linalg.norm(n, axis=-1) > 0.5
    assert ok.mean() > 0.8
    c, r = np.meshgrid(np.arange(128.0), np.arange(32.0))
    pts = P.unproject(cam, np.stack([c, r], axis=-1), depth)
    err = np.linalg.norm(n[2:-2, 2:-2] + pts[2:-2, 2:-2] / 5.0, axis=-1)
    assert err.max() < 1e-2


def test_tilted_plane_normals_face_observer():
    cam = _pinhole()
    c, r = np.meshgrid(np.arange(64.0), np.arange(48.0))
    depth = 2.0 / (1.0 - 0.3 * (c - cam.cx) / cam.fx)
    depth += np.random.default_rng(31).normal(0.0, 1e-4, depth.shape)
    n = P.estimate_normals(depth, cam)
    ok = np.linalg.norm(n, axis=-1) > 0.5
    pts = P.unproject(cam, np.stack([c, r], axis=-1), depth)
    assert ok.any()
    assert (np.einsum("ij,ij->i", n[ok], pts[ok]) < 0).all()


def test_normal_config_radius_changes_support():
    # A three-pixel-wide valid stripe: 1x1 windows (radius 0) hold one point,
    # the default radius-2 windows hold 15 coplanar points.
    cam = _pinhole()
    depth = np.zeros((48, 64))
    depth[:, 30:33] = 2.0
    narrow = P.estimate_normals(depth, cam, P.NormalConfig(radius_min=0.0, radius_max=0.0))
    assert not narrow.any()
    wide = P.estimate_normals(depth, cam)
    ok = np.linalg.norm(wide, axis=-1) > 0.5
    assert ok[:, 30:33].all() and not ok[:, :30].any()


def test_constant_pyramid_is_constant():
    cam = _pinhole()
    pyr = P.build_pyramid(np.full((48, 64), 0.37), np.full((48, 64), 2.0), cam, (0.25, 0.5, 1.0))
    for lvl in pyr.levels:
        assert np.allclose(lvl.intensity, 0.37) and np.allclose(lvl.depth, 2.0)


def test_level_sizes_740x460():
    cam = Intrinsics(400.0, 400.0, 370.0, 230.0, 740, 460, P.PINHOLE, 0.1, 50.0)
    img = np.full((460, 740), 0.5)
    pyr = P.build_pyramid(img, np.full((460, 740), 2.0), cam)
    assert [l.shape for l in pyr.levels] == [(57, 92), (115, 185), (230, 370)]
    assert [(l.intrinsics.width, l.intrinsics.height) for l in pyr.levels] == [
        (92, 57), (185, 115), (370, 230)]


@pytest.mark.parametrize("scales", [(), (0.5, 0.25), (0.5, 1.5), (0.0,)])
def test_bad_scales_rejected(scales):
    img = np.full((12, 16), 0.5)
    with pytest.raises(P.PyramidConfigError):
        P.build_pyramid(img, img, _pinhole(16, 12, 20.0), scales=scales)


def test_shape_mismatch_rejected():
    with pytest.raises(ValueError):
        P.build_pyramid(np.zeros((12, 16)), np.ones((12, 15)), _pinhole(16, 12, 20.0), (0.5,))


def test_depth_median_never_blends_and_matches_bruteforce():
    rng = np.random.default_rng(32)
    cam = _pinhole(15, 11, 20.0)
    depth = rng.uniform(1.0, 5.0, (11, 15))
    depth[rng.random((11, 15)) < 0.3] = 0.0
    s = 1.0 / 3.0
    lvl = P.build_pyramid(rng.random((11, 15)), depth, cam, (s,)).levels[0]
    for r in range(lvl.shape[0]):
        for c in range(lvl.shape[1]):
            members = sorted(depth[rr, cc] for rr in range(11) for cc in range(15)
                             if math.floor(rr * s) == r and math.floor(cc * s) == c
                             and depth[rr, cc] > 0)
            want = members[(len(members) - 1) // 2] if members else 0.0
            assert lvl.depth[r, c] == want


def test_pyramid_normals_unit_or_zero():
    cam = _pinhole()
    pyr = P.build_pyramid(np.full((48, 64), 0.5), np.full((48, 64), 2.0), cam, (0.25, 0.5))
    for lvl in pyr.levels:
        nn = np.linalg.norm(lvl.normals, axis=-1)
        assert np.all((np.abs(nn - 1.0) < 1e-6) | (nn == 0.0))
        assert np.all(lvl.normal_valid <= lvl.depth_valid)


def test_build_cue_image_uses_given_normals():
    cam = _pinhole(16, 12, 20.0)
    n = np.zeros((12, 16, 3))
    n[..., 2] = -1.0
    img = P.build_cue_image(np.full((12, 16), 0.5), np.full((12, 16), 1.0), cam, normals=n)
    np.testing.assert_array_equal(img.normals, n)
    est = P.build_cue_image(np.full((12, 16), 0.5), np.full((12, 16), 1.0), cam)
    np.testing.assert_array_equal(est.normals, P.estimate_normals(np.full((12, 16), 1.0), cam))
