"""Dataset I/O against a dataset directory written
by the reference's generate_synthetic (tests/golden/dataset.npz, made by
tests/golden/make_golden.py) and the reference's test cases
(pkg/tests/test_dataset_io.py:61-205)."""

import numpy as np
import pytest

import paper_2303_16878_b200 as P
from paper_2303_16878_b200 import dataset as DS
from paper_2303_16878_b200.camera import Intrinsics, SensorExtrinsics
from tests.fixtures import GOLDEN


def unpack(tmp_path):
    z = np.load(GOLDEN / "dataset.npz")
    root = tmp_path / "ds"
    for k, rel in enumerate(z["files"]):
        p = root / str(rel)
        p.parent.mkdir(parents=True, exist_ok=True)
        p.write_bytes(z[f"file_{k}"].tobytes())
    return root, z


def test_host_load_matches_reference_bit_exact(tmp_path):
    root, z = unpack(tmp_path)
    manifest, guess, frames = DS.load_dataset(root)
    assert [s.sensor_id for s in manifest.sensors] == ["cam0", "lidar0"]
    np.testing.assert_array_equal(guess.timestamps, z["stamps"])
    np.testing.assert_array_equal(np.stack([p.as_row() for p in guess.poses]), z["guess"])
    for sid, nodes in frames.items():
        assert len(nodes) == 3
        for f, node in enumerate(nodes):
            assert node.sensor_id == sid and node.timestamp == z["stamps"][f]
            for l, img in enumerate(node.pyramid.levels):
                key = f"{sid}_I_{f}_{l}"
                if key not in z.files:
                    continue
                np.testing.assert_array_equal(img.intensity, z[key])
                np.testing.assert_array_equal(img.depth, z[f"{sid}_D_{f}_{l}"])
                np.testing.assert_array_equal(img.normals, z[f"{sid}_N_{f}_{l}"])


def test_writers_reproduce_reference_files_byte_for_byte(tmp_path):
    root, z = unpack(tmp_path)
    manifest = DS.load_manifest(root / "manifest")
    out = tmp_path / "out"
    out.mkdir()
    DS.save_manifest(manifest, out / "manifest")
    assert (out / "manifest").read_bytes() == (root / "manifest").read_bytes()
    for name in ("trajectory.txt", "trajectory_gt.txt"):
        DS.save_trajectory(DS.load_trajectory(root / name), out / name)
        assert (out / name).read_bytes() == (root / name).read_bytes()
    for s in manifest.sensors:
        for f in sorted((root / s.intensity_dir).iterdir()):
            DS.write_intensity(out / "i.pgm", DS.read_intensity(f))
            assert (out / "i.pgm").read_bytes() == f.read_bytes()
        for f in sorted((root / s.depth_dir).iterdir()):
            DS.write_depth(out / "d.pgm", DS.read_depth(f, s.depth_scale), s.depth_scale)
            assert (out / "d.pgm").read_bytes() == f.read_bytes()


def test_raster_round_trips(tmp_path):
    rng = np.random.default_rng(61)
    a16 = rng.integers(0, 65536, (7, 9)).astype(np.uint16)
    DS.write_raster(tmp_path / "a.pgm", a16)
    b = DS.read_raster(tmp_path / "a.pgm")
    assert b.dtype == np.uint16 and np.array_equal(a16, b)
    a8 = rng.integers(0, 256, (5, 3)).astype(np.uint8)
    DS.write_raster(tmp_path / "b.pgm", a8)
    b = DS.read_raster(tmp_path / "b.pgm")
    assert b.dtype == np.uint8 and np.array_equal(a8, b)
    with pytest.raises(ValueError):
        DS.write_raster(tmp_path / "c.pgm", a16.astype(np.int32))


def test_header_comments_and_errors(tmp_path):
    payload = np.arange(6, dtype=">u2").tobytes()
    (tmp_path / "c.pgm").write_bytes(b"P5\n# a comment\n3 2\n# another\n65535\n" + payload)
    assert np.array_equal(DS.read_raster(tmp_path / "c.pgm"), np.arange(6).reshape(2, 3))
    (tmp_path / "t.pgm").write_bytes(b"P5\n3 2\n65535\n" + payload[:-1])
    with pytest.raises(DS.DatasetError):
        DS.read_raster(tmp_path / "t.pgm")
    (tmp_path / "p2.pgm").write_bytes(b"P2\n3 2\n255\n0 1 2 3 4 5\n")
    with pytest.raises(DS.DatasetError):
        DS.read_raster(tmp_path / "p2.pgm")
    with pytest.raises(DS.MissingFileError):
        DS.read_raster(tmp_path / "missing.pgm")


def test_intensity_and_depth_semantics(tmp_path):
    v = np.array([[0.0, 0.25, 1.0], [0.5, 0.999, 1.2]])
    DS.write_intensity(tmp_path / "i.pgm", v)
    assert np.abs(DS.read_intensity(tmp_path / "i.pgm") - np.clip(v, 0, 1)).max() <= 0.5 / 65535
    DS.write_raster(tmp_path / "i8.pgm", np.array([[0, 255, 51]], dtype=np.uint8))
    assert np.array_equal(DS.read_intensity(tmp_path / "i8.pgm"), [[0.0, 1.0, 0.2]])
    m = np.array([[0.0, 1.234, np.nan], [-1.0, 70.0, 0.0004]])
    DS.write_depth(tmp_path / "d.pgm", m, 0.001)
    raw = DS.read_raster(tmp_path / "d.pgm")
    assert raw.tolist() == [[0, 1234, 0], [0, 65535, 1]]
    np.testing.assert_array_equal(DS.read_depth(tmp_path / "d.pgm", 0.001), raw * 0.001)
    with pytest.raises(DS.DatasetError):
        DS.read_depth(tmp_path / "i8.pgm", 0.001)


def test_trajectory_parsing(tmp_path):
    poses = [P.Pose.from_quat([1.0, 2.0, 3.0], [0.0, 0.0, np.sin(0.1), np.cos(0.1)]),
             P.Pose.identity()]
    tr = DS.Trajectory([0.5, 1.5], poses)
    DS.save_trajectory(tr, tmp_path / "t.txt")
    back = DS.load_trajectory(tmp_path / "t.txt")
    assert np.allclose(back.timestamps, tr.timestamps)
    for a, b in zip(back.poses, tr.poses):
        assert np.allclose(a.rotation, b.rotation, atol=1e-9)
        assert np.allclose(a.translation, b.translation, atol=1e-9)
    (tmp_path / "c.txt").write_text("# header\n\n0.0 0 0 0 0 0 0 1\n  # x\n1.0 0 0 0 0 0 0 1\n")
    assert len(DS.load_trajectory(tmp_path / "c.txt")) == 2
    (tmp_path / "o.txt").write_text("1.0 0 0 0 0 0 0 1\n0.5 0 0 0 0 0 0 1\n")
    with pytest.raises(DS.TrajectoryFormatError):
        DS.load_trajectory(tmp_path / "o.txt")
    (tmp_path / "m.txt").write_text("0.0 0 0 0 0 0 0 1\n1.0 0 0 0 0 0 1\n")
    with pytest.raises(DS.TrajectoryFormatError, match=":2:"):
        DS.load_trajectory(tmp_path / "m.txt")
    (tmp_path / "e.txt").write_text("# nothing\n")
    with pytest.raises(DS.TrajectoryFormatError):
        DS.load_trajectory(tmp_path / "e.txt")


def test_manifest_round_trip_and_errors(tmp_path):
    cam = Intrinsics(70.0, 70.0, 80.0, 60.0, 160, 120, P.PINHOLE, 0.1, 50.0)
    m = DS.DatasetManifest([DS.SensorConfig("cam0", cam, SensorExtrinsics.identity(), 0.001,
                                            "cam0/intensity", "cam0/depth")],
                           pyramid_scales=(0.25, 0.5))
    DS.save_manifest(m, tmp_path / "manifest")
    back = DS.load_manifest(tmp_path / "manifest")
    assert back.sensors[0].intrinsics == cam and back.pyramid_scales == (0.25, 0.5)
    with pytest.raises(DS.ManifestError):
        DS.SensorConfig("x", cam, SensorExtrinsics.identity(), 0.0, "i", "d")
    (tmp_path / "bad").write_text("{not json")
    with pytest.raises(DS.ManifestError):
        DS.load_manifest(tmp_path / "bad")
    (tmp_path / "bad2").write_text('{"sensors": [{"sensor_id": "a"}]}')
    with pytest.raises(DS.ManifestError):
        DS.load_manifest(tmp_path / "bad2")
    with pytest.raises(DS.MissingFileError):
        DS.load_manifest(tmp_path / "none")


def test_load_dataset_missing_and_mismatched_images(tmp_path):
    root, z = unpack(tmp_path)
    stamps = z["stamps"]
    (root / "cam0" / "depth" / f"{stamps[1]:.6f}.pgm").unlink()
    with pytest.raises(DS.MissingFileError, match="cam0"):
        DS.load_dataset(root)
    root2, _ = unpack(tmp_path / "b")
    DS.write_intensity(root2 / "cam0" / "intensity" / f"{stamps[0]:.6f}.pgm", np.zeros((10, 10)))
    with pytest.raises(DS.DimensionMismatchError):
        DS.load_dataset(root2)


def test_write_dataset_round_trip(tmp_path):
    cam = Intrinsics(20.0, 20.0, 8.0, 6.0, 16, 12, P.PINHOLE, 0.1, 50.0)
    rng = np.random.default_rng(3)
    frames = [(rng.random((12, 16)), rng.uniform(0.5, 3.0, (12, 16))) for _ in range(2)]
    m = DS.DatasetManifest([DS.SensorConfig("c", cam, SensorExtrinsics.identity(), 0.001,
                                            "c/intensity", "c/depth")], pyramid_scales=(0.5, 1.0))
    tr = DS.Trajectory([0.0, 0.1], [P.Pose.identity(), P.Pose.identity()])
    DS.write_dataset(tmp_path / "w", m, tr, {"c": frames})
    _, _, got = DS.load_dataset(tmp_path / "w")
    lvl = got["c"][1].pyramid.levels[-1]
    assert np.abs(lvl.intensity - frames[1][0]).max() <= 0.5 / 65535
    assert np.abs(lvl.depth - frames[1][1]).max() <= 0.0005 + 1e-12
