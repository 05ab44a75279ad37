"""GPU cue-pyramid builder (K6, csrc/pyramid.cu) against the reference's own
outputs (tests/golden/pyramid.npz) and the host restatement (cueimage.py,
itself bit-exact to the reference — tests/test_pyramid.py).

Bars: downscaled intensity / depth and the downscale of given normals are
bit-exact; estimated normals have bit-exact validity and agree to 1e-9 per
component (1e-10 against the host restatement) — the 3x3 eigenproblem is
Jacobi here, LAPACK in the reference, and the pixels where the two could
decide differently are re-decided with eigh on the host."""
import math

import numpy as np
import pytest

import paper_2303_16878_b200 as P
from paper_2303_16878_b200.camera import Intrinsics
from paper_2303_16878_b200.cueimage import downscale_cues
from tests.fixtures import GOLDEN

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

NORMAL_TOL = 1e-9


def _cam(row):
    model = P.PINHOLE if row[6] == 0 else P.SPHERICAL
    return Intrinsics(row[0], row[1], row[2], row[3], int(row[4]), int(row[5]), model, row[7],
                      row[8])


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN / "pyramid.npz")


def _valid(n):
    return np.linalg.norm(n, axis=-1) > 0.5


@pytest.mark.parametrize("tag", ["p", "s"])
def test_device_normals_match_reference(golden, tag):
    cam = _cam(golden[f"{tag}_cam"])
    ref = golden[f"{tag}_normals"]
    n = P.estimate_normals_device(torch.from_numpy(golden[f"{tag}_D"]).cuda(), cam)
    n = n.cpu().numpy()
    assert np.array_equal(_valid(n), _valid(ref))
    assert np.abs(n - ref).max() <= NORMAL_TOL


@pytest.mark.parametrize("tag", ["p", "s"])
def test_device_pyramid_matches_reference(golden, tag):
    cam = _cam(golden[f"{tag}_cam"])
    scales = tuple(golden[f"{tag}_scales"])
    pyr = P.build_pyramid(golden[f"{tag}_I"], golden[f"{tag}_D"], cam, scales, device="cuda")
    assert pyr.scales == scales
    for l, img in enumerate(pyr.levels):
        assert isinstance(img, P.DeviceCueImage)
        assert img.intrinsics == cam.scaled(scales[l])
        np.testing.assert_array_equal(img.device_intensity.cpu().numpy(), golden[f"{tag}_I_{l}"])
        np.testing.assert_array_equal(img.device_depth.cpu().numpy(), golden[f"{tag}_D_{l}"])
        n = img.device_normals.cpu().numpy()
        assert np.array_equal(_valid(n), _valid(golden[f"{tag}_N_{l}"]))
        assert np.abs(n - golden[f"{tag}_N_{l}"]).max() <= NORMAL_TOL


@pytest.mark.parametrize("s", [1.0, 0.5, 0.25, 0.125, 1.0 / 3.0, 0.3])
def test_device_downscale_bit_exact(s):
    rng = np.random.default_rng(int(s * 1000))
    H, W = 37, 53
    cam = Intrinsics(40.0, 40.0, W / 2, H / 2, W, H, P.PINHOLE, 0.1, 20.0)
    inten = rng.random((H, W))
    depth = rng.uniform(0.05, 25.0, (H, W))  # some below / above range
    depth[rng.random((H, W)) < 0.2] = 0.0
    depth[rng.random((H, W)) < 0.02] = 7.5  # ties for the median
    normals = rng.normal(size=(H, W, 3))
    normals /= np.linalg.norm(normals, axis=-1, keepdims=True)
    normals[rng.random((H, W)) < 0.3] = 0.0
    normals[rng.random((H, W)) < 0.1] *= 0.7  # non-unit but valid
    want = downscale_cues(inten, depth, normals, (depth >= 0.1) & (depth <= 20.0),
                          np.linalg.norm(normals, axis=-1) > 0.5, s)
    from paper_2303_16878_b200.pyramid_device import downscale_cues_device
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a[None])).cuda()  # noqa: E731
    got = downscale_cues_device(T(inten), T(depth), T(normals), cam, s)
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g[0].cpu().numpy(), w)


def test_device_pyramid_batch_equals_single():
    from paper_2303_16878_b200 import scenes as S

    cam = S.rgbd_160()
    poses = S.room_loop(3)
    rows = S.sensor_rows(poses, P.Pose.identity()).cuda()
    inten, depth, _ = S.render_batch(S.BoxScene(), cam, rows)
    batch = P.build_pyramids_device(inten, depth, cam, (0.25, 0.5, 1.0))
    for b in range(3):
        one = P.build_pyramid(inten[b], depth[b], cam, (0.25, 0.5, 1.0), device="cuda")
        for x, y in zip(batch[b].levels, one.levels):
            assert torch.equal(x.device_intensity, y.device_intensity)
            assert torch.equal(x.device_depth, y.device_depth)
            assert torch.equal(x.device_normals, y.device_normals)


def test_batched_texel_build_equals_per_frame():
    """FrameStore.prefetch builds the texels of consecutive frames of one
    device batch with one pba_build_texels_batch call; per-frame
    pba_build_texels gives the same bytes (and host cue images still take
    the per-frame path)."""
    from paper_2303_16878_b200 import scenes as S
    from paper_2303_16878_b200.device import FrameStore

    cam = S.rgbd_160()
    rows = S.sensor_rows(S.room_loop(5), P.Pose.identity()).cuda()
    inten, depth, _ = S.render_batch(S.BoxScene(), cam, rows)
    pyrs = P.build_pyramids_device(inten, depth, cam, (0.5, 1.0))
    dev = torch.device("cuda", 0)
    for level in (0, 1):
        cues = [p.levels[level] for p in pyrs]
        batched, single = FrameStore(dev), FrameStore(dev)
        batched.prefetch(cues)
        assert FrameStore._batch_run(cues, 0, cues[0].shape[0] * cues[0].shape[1]) == 5
        for cue in cues:
            tb, mb, rb, cb = batched.frame(cue)
            ts, ms, rs, cs = single.frame(cue)
            assert torch.equal(tb, ts) and torch.equal(mb, ms) and torch.equal(rb, rs)
            assert bytes(cb) == bytes(cs)


def _assert_normals_equal_host(depth_batch, cam, dev):
    """zero validity flips, normals within 1e-10, against the host
    restatement (bit-exact to the reference's estimate_normals)."""
    worst = 0.0
    for b in range(depth_batch.shape[0]):
        host = P.estimate_normals(depth_batch[b], cam)
        vh, vd = _valid(host), _valid(dev[b])
        assert np.array_equal(vh, vd), int((vh != vd).sum())
        if vh.any():
            worst = max(worst, float(np.abs(host[vh] - dev[b][vh]).max()))
    assert worst <= 1e-10, worst
    return worst


def test_device_normals_on_lidar_scans_match_host():
    """OS0-128 scans along the c4 corridor: validity bit-exact."""
    from paper_2303_16878_b200 import scenes as S
    from paper_2303_16878_b200 import pyramid_device as PD

    cam = S.lidar_os0_128()
    poses = S.perturb(S.corridor_trajectory(12, 2.0), 0.05, math.radians(2.0), 3)
    rows = S.sensor_rows(poses, P.Pose(np.eye(3), [0.0, 0.0, -0.05])).cuda()
    _, depth, _ = S.render_batch(S.corridor_scene(40.0), cam, rows)
    dev = P.estimate_normals_device(depth, cam).cpu().numpy()
    _assert_normals_equal_host(depth.cpu().numpy(), cam, dev)
    assert PD.last_recheck_count >= 0


def test_device_normals_on_rgbd_scans_match_host():
    """640x480 forward-looking RGB-D frames (c3 / c5 mount): validity bit-exact."""
    import bench
    from paper_2303_16878_b200 import scenes as S

    cam = S.tum_640()
    poses = S.perturb(S.corridor_trajectory(6, 0.3), 0.05, math.radians(2.0), 5)
    rows = S.sensor_rows(poses, P.Pose(bench.FORWARD_CAMERA, [0.0, 0.0, 0.1])).cuda()
    _, depth, _ = S.render_batch(S.corridor_scene(30.0), cam, rows)
    dev = P.estimate_normals_device(depth, cam).cpu().numpy()
    _assert_normals_equal_host(depth.cpu().numpy(), cam, dev)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_device_normals_knife_edge_inputs_rechecked(seed):
    """Depth images built to sit on the gates: planes with noise at many
    scales (near-degenerate scatter), line-like strips, grazing views and
    holes — and, for each image, NormalConfigs whose degeneracy ratio is set
    to the exact eigenvalue ratio lam1 / lam2 of chosen pixels, so those
    pixels' planarity test is decided by the last bits of the eigensolver.
    The device must hand them to the host's eigh: zero validity flips,
    including with a tiny first recheck buffer (the grow-and-rerun path)."""
    from paper_2303_16878_b200 import pyramid_device as PD
    from paper_2303_16878_b200.cueimage import NormalConfig, window_scatter

    rng = np.random.default_rng(seed)
    H, W = 48, 64
    cam = Intrinsics(60.0, 60.0, W / 2, H / 2, W, H, P.PINHOLE, 0.1, 20.0)
    cols, rows = np.meshgrid(np.arange(W, dtype=float), np.arange(H, dtype=float))
    batch = []
    for k in range(6):
        base = 2.0 + 0.02 * k * cols + 0.001 * rows  # tilted plane (grazing for large k)
        noise = rng.normal(size=(H, W)) * 10.0 ** rng.uniform(-14, -2, (H, W))
        d = base + noise
        if k % 3 == 1:  # a thin strip: line-like windows
            d[:, :] = 0.0
            d[H // 2, :] = base[H // 2, :]
            d[H // 2 + 1, ::7] = base[H // 2 + 1, ::7]
        if k % 3 == 2:
            d[rng.random((H, W)) < 0.3] = 0.0
        batch.append(d)
    depth = np.stack(batch)
    _, _, S, _ = window_scatter(depth[0], cam, NormalConfig())
    lam = np.linalg.eigvalsh(S)
    ratio = lam[:, 1] / lam[:, 2]
    picks = rng.choice(np.nonzero((ratio > 1e-6) & (ratio < 0.5))[0], 3, replace=False)
    rechecked = 0
    for cfg in [NormalConfig()] + [NormalConfig(degeneracy_ratio=float(ratio[i])) for i in picks]:
        dev = P.estimate_normals_device(torch.from_numpy(depth).cuda(), cam, cfg,
                                        recheck_capacity=1).cpu().numpy()
        for b in range(depth.shape[0]):
            host = P.estimate_normals(depth[b], cam, cfg)
            assert np.array_equal(_valid(host), _valid(dev[b]))
            vh = _valid(host)
            if vh.any():
                assert np.abs(host[vh] - dev[b][vh]).max() <= 1e-10
        rechecked += PD.last_recheck_count
    assert rechecked > 0  # the host path was exercised


@pytest.mark.parametrize("config", ["c4", "c5"])
def test_bench_input_pyramids_match_host_builder(config):
    """The bench's own inputs (bench.build_problem: renders -> K6): every
    level of the device pyramids against the host build_pyramid of the same
    finest-level intensity / depth — intensity, depth bit-exact, normal
    validity bit-exact, normals within 1e-10."""
    import bench

    problems, _, _, meta = bench.build_problem(config, torch.device("cuda", 0), 4)
    for prob in problems:
        for node in prob.graph.nodes:
            pyr = node.pyramid
            fin = pyr.levels[-1]
            inten = fin.device_intensity.cpu().numpy()
            depth = fin.device_depth.cpu().numpy()
            host = P.build_pyramid(inten, depth, fin.intrinsics, pyr.scales)
            for h, d in zip(host.levels, pyr.levels):
                np.testing.assert_array_equal(d.device_intensity.cpu().numpy(), h.intensity)
                np.testing.assert_array_equal(d.device_depth.cpu().numpy(), h.depth)
                n = d.device_normals.cpu().numpy()
                assert np.array_equal(_valid(n), _valid(h.normals))
                assert np.abs(n - h.normals).max() <= 1e-10


def test_device_pyramid_errors():
    cam = Intrinsics(20.0, 20.0, 8.0, 6.0, 16, 12, P.PINHOLE, 0.1, 10.0)
    img = np.full((12, 16), 0.5)
    with pytest.raises(P.PyramidConfigError):
        P.build_pyramid(img, img, cam, (0.5, 0.25), device="cuda")
    with pytest.raises(ValueError):
        P.build_pyramid(img, np.ones((12, 15)), cam, (0.5,), device="cuda")
    with pytest.raises(ValueError):
        P.estimate_normals_device(np.ones((11, 16)), cam)


def test_device_empty_depth_gives_zero_normals():
    cam = Intrinsics(20.0, 20.0, 8.0, 6.0, 16, 12, P.PINHOLE, 0.1, 10.0)
    n = P.estimate_normals_device(np.full((12, 16), math.nan), cam)
    assert n.shape == (12, 16, 3) and not bool(n.any())


def test_device_load_dataset_matches_reference(tmp_path):
    from paper_2303_16878_b200 import dataset as DS
    from tests.test_dataset import unpack

    root, z = unpack(tmp_path)
    _, guess, frames = DS.load_dataset(root, device="cuda")
    np.testing.assert_array_equal(guess.timestamps, z["stamps"])
    checked = 0
    for sid, nodes in frames.items():
        for f, node in enumerate(nodes):
            for l, img in enumerate(node.pyramid.levels):
                key = f"{sid}_I_{f}_{l}"
                if key not in z.files:
                    continue
                assert isinstance(img, P.DeviceCueImage)
                np.testing.assert_array_equal(img.device_intensity.cpu().numpy(), z[key])
                np.testing.assert_array_equal(img.device_depth.cpu().numpy(), z[f"{sid}_D_{f}_{l}"])
                n = img.device_normals.cpu().numpy()
                ref = z[f"{sid}_N_{f}_{l}"]
                assert np.array_equal(_valid(n), _valid(ref))
                assert np.abs(n - ref).max() <= NORMAL_TOL
                checked += 1
    assert checked == 2 * (3 + 2)


def test_device_raster_decode_kinds():
    from paper_2303_16878_b200 import native as N

    lib = N.load()
    vals = np.array([0, 1, 255, 256, 4660, 65535], dtype=">u2")
    raw = torch.from_numpy(np.frombuffer(vals.tobytes(), dtype=np.uint8).copy()).cuda()
    out = torch.empty(6, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    N.check(lib.pba_decode_raster(raw.data_ptr(), 6, N.PBA_RASTER_U16_DEPTH, 0.001,
                                  out.data_ptr(), stream), "decode")
    np.testing.assert_array_equal(out.cpu().numpy(), vals.astype(np.uint16).astype(float) * 0.001)
    N.check(lib.pba_decode_raster(raw.data_ptr(), 6, N.PBA_RASTER_U16_INTENSITY, 0.0,
                                  out.data_ptr(), stream), "decode")
    np.testing.assert_array_equal(out.cpu().numpy(), vals.astype(np.uint16).astype(float) / 65535.0)
    N.check(lib.pba_decode_raster(raw.data_ptr(), 6, N.PBA_RASTER_U8_INTENSITY, 0.0,
                                  out.data_ptr(), stream), "decode")
    b = raw.cpu().numpy()[:6].astype(float) / 255.0
    np.testing.assert_array_equal(out.cpu().numpy(), b)
    assert lib.pba_decode_raster(raw.data_ptr(), 6, 7, 0.0, out.data_ptr(), stream) != 0


def test_pipeline_from_disk_on_device_matches_host_pipeline(tmp_path):
    """load_dataset -> build_graph -> solve_hierarchical -> evaluate_ate, all
    GPU options on, against the same pipeline on host-built pyramids."""
    from paper_2303_16878_b200 import dataset as DS
    from tests.test_dataset import unpack

    root, _ = unpack(tmp_path)
    gt = DS.load_trajectory(root / "trajectory_gt.txt")
    results = []
    for device in (None, "cuda"):
        manifest, guess, frames = DS.load_dataset(root, device=device)
        ext = manifest.sensors[0].extrinsics
        graph = P.build_graph(frames["cam0"], extrinsics=ext, device=device)
        prob = P.BAProblem(graph, {"cam0": ext})
        res = P.solve_hierarchical(prob, P.SolverConfig())
        rep = P.evaluate_ate(P.trajectory_from_poses(guess.timestamps, res.poses), gt)
        results.append((graph.edge_pairs(), res, rep))
    (e_h, r_h, a_h), (e_d, r_d, a_d) = results
    assert e_h == e_d
    assert [(r.level, r.iteration, r.accepted, r.valid_blocks) for r in r_h.records] == \
        [(r.level, r.iteration, r.accepted, r.valid_blocks) for r in r_d.records]
    for p, q in zip(r_h.poses, r_d.poses):
        assert np.abs(p.translation - q.translation).max() < 1e-9
    assert abs(a_h.rmse - a_d.rmse) < 1e-9
