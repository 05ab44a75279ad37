"""Host-side logic (CPU): drop-in types vs reference semantics, bit-exact
pair lists and pyramid indices, and the C ABI library surface."""
import ctypes
import math
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2303_16878_b200 as P
from paper_2303_16878_b200 import native
from oracle import oracle as O
from tests import fixtures as F

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("name", ["pinhole_small", "spherical_small"])
def test_cueimage_derivation_bit_exact(name):
    d = F.load(name)
    pyrs = F.pyramids(d)
    for f, pyr in enumerate(pyrs):
        for l, img in enumerate(pyr.levels):
            assert np.array_equal(F.mask_bits(img), d[f"M_{f}_{l}"])
            if f == 0:
                g = np.concatenate([img.grad_intensity.reshape(-1), img.grad_depth.reshape(-1),
                                    img.grad_normals.reshape(-1)])
                assert np.array_equal(g, d[f"G_{f}_{l}"])


def test_footprint_index_bit_exact():
    d = F.load("footprint")
    k = 0
    while f"fp_{k}" in d:
        h, w, s, oh, ow = d[f"fp_{k}"]
        idx, keep, out_h, out_w = P.footprint_index(int(h), int(w), float(s))
        assert (out_h, out_w) == (int(oh), int(ow))
        rows = np.where(keep[:, 0], idx[:, 0] // max(out_w, 1), -1)
        cols = np.where(keep[0, :], idx[0, :] % max(out_w, 1), -1)
        assert np.array_equal(rows, d[f"fp_rows_{k}"])
        assert np.array_equal(cols, d[f"fp_cols_{k}"])
        assert [int(idx[keep].sum()), int(keep.sum())] == list(d[f"fp_sum_{k}"])
        k += 1


@pytest.mark.parametrize("name", ["pinhole_small", "spherical_small"])
def test_build_graph_matches_reference_edge_list(name):
    d = F.load(name)
    pyrs = F.pyramids(d)
    guess = F.poses(d["guess"])
    nodes = [P.FrameNode(k, guess[k], pyrs[k], 0.1 * k) for k in range(len(pyrs))]
    ext = P.SensorExtrinsics(P.Pose.from_row(d["ext"]))
    g = P.build_graph(nodes, extrinsics=ext)
    assert [(e.i, e.j) for e in g.edges] == [tuple(map(int, e)) for e in d["edges"]]
    assert [e.kind == P.COVISIBILITY for e in g.edges] == list(d["edge_kinds"])
    g2 = P.build_graph(nodes, extrinsics=ext, threads=4)
    assert g2.edges == g.edges


def test_build_graph_validation():
    cam = P.Intrinsics(20, 20, 8, 6, 16, 12, P.PINHOLE, 0.1, 10.0)
    img = P.CueImage(np.full((12, 16), 0.5), np.full((12, 16), 2.0), np.zeros((12, 16, 3)), cam)
    pyr = P.CuePyramid((img,), (1.0,))
    n0 = P.FrameNode(0, P.Pose.identity(), pyr, 0.0)
    with pytest.raises(P.GraphConfigError):
        P.build_graph([n0])
    with pytest.raises(P.GraphConfigError):
        P.build_graph([n0, P.FrameNode(0, P.Pose.identity(), pyr, 0.1)])
    with pytest.raises(P.GraphConfigError):
        P.build_graph([n0, P.FrameNode(1, P.Pose.identity(), pyr, -1.0)])


def test_boxplus_matches_oracle_and_sign_convention():
    rng = np.random.default_rng(3)
    for _ in range(50):
        x = P.exp(P.PerturbationVector(rng.uniform(-1, 1, 3), rng.uniform(-0.3, 0.3, 3)))
        v = np.concatenate([rng.uniform(-0.2, 0.2, 3), rng.uniform(-0.2, 0.2, 3)])
        y = P.boxplus(x, P.PerturbationVector.from_vector(v))
        R2, t2, g2 = O.boxplus(x.rotation, x.translation, x.generation, v)
        assert np.array_equal(y.rotation, R2) and np.array_equal(y.translation, t2)
        assert y.generation == g2 == 1
    # d(exp(v) p)/d v_rot = -2 [p]x at v = 0 (Hamilton; reference test_geometry.py:183-197)
    p = np.array([0.3, -1.2, 2.0])
    h = 1e-7
    jac = np.zeros((3, 3))
    for k in range(3):
        e = np.zeros(3); e[k] = h
        jac[:, k] = (P.exp(P.PerturbationVector(np.zeros(3), e)).transform(p)
                     - P.exp(P.PerturbationVector(np.zeros(3), -e)).transform(p)) / (2 * h)
    assert np.allclose(jac, -2.0 * P.skew(p), atol=1e-6)
    with pytest.raises(P.InvalidPerturbationError):
        P.exp(P.PerturbationVector(np.zeros(3), [0.8, 0.6, 0.1]))


def test_reorthonormalisation_after_1000_compositions():
    x = P.Pose.identity()
    v = P.PerturbationVector([0.001, 0, 0], [0.001, 0.002, -0.001])
    for _ in range(999):
        x = P.boxplus(x, v)
    assert x.generation == 999
    x = P.boxplus(x, v)
    assert x.generation == 0
    assert np.allclose(x.rotation @ x.rotation.T, np.eye(3), atol=1e-15)


def test_intrinsics_scaled_half_pixel_rule():
    cam = P.Intrinsics(400.0, 400.0, 370.0, 230.0, 740, 460, P.PINHOLE, 0.1, 50.0)
    dims = [(cam.scaled(s).height, cam.scaled(s).width) for s in (0.125, 0.25, 0.5)]
    assert dims == [(57, 92), (115, 185), (230, 370)]
    s = 0.25
    assert cam.scaled(s).cx == 370.0 * s + (s - 1) / 2


def test_solver_config_validation_and_defaults():
    cfg = P.SolverConfig()
    assert list(cfg.omega_diagonal()) == [1.0, 10.0, 1.0, 1.0, 1.0]
    with pytest.raises(ValueError):
        P.SolverConfig(huber_delta_depth=0.0)
    with pytest.raises(ValueError):
        P.SolverConfig(termination_rel_decrease=1.0)
    with pytest.raises(ValueError):
        P.SolverConfig(pixel_stride=0)
    assert cfg.linear_solver == "cholesky"
    with pytest.raises(ValueError):
        P.SolverConfig(linear_solver="lu")
    with pytest.raises(ValueError):
        P.SolverConfig(linear_solver="pcg", pcg_max_iterations=0)


def test_pcg_block_rows_pattern():
    from paper_2303_16878_b200.device import block_rows

    rng = np.random.default_rng(2)
    n = 30
    slot = np.array([-1 if k == 4 else k - (k > 4) for k in range(n)], np.int32)
    pi = rng.integers(0, n, 200).astype(np.int32)
    pj = (pi + rng.integers(1, n, 200)) % n
    pj = pj.astype(np.int32)
    row_ptr, cols = block_rows(slot, pi, pj)
    dense = np.eye(n - 1, dtype=bool)
    for a, b in zip(slot[pi], slot[pj]):
        if a >= 0 and b >= 0:
            dense[a, b] = dense[b, a] = True
    for r in range(n - 1):
        got = cols[row_ptr[r]: row_ptr[r + 1]]
        assert list(got) == list(np.nonzero(dense[r])[0])  # ascending, diagonal included


def test_check_connectivity_names_stranded_pose():
    d = F.load("pinhole_small")
    prob, _ = F.single_problem(d)
    prob.graph.edges = [e for e in prob.graph.edges if 3 not in (e.i, e.j)]
    with pytest.raises(P.UnderConstrainedError, match="3"):
        P.check_connectivity([prob])


def _header_functions():
    text = (ROOT / "include" / "pba.h").read_text()
    return sorted(set(re.findall(r"\b(pba_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = native.load()
    names = _header_functions()
    assert set(names) == set(native.EXPORTED)
    for name in names:
        assert hasattr(lib, name), name
    assert lib.pba_texel_bytes() == 128
    assert b"sm_100a" in lib.pba_version()


def test_host_planning_functions():
    lib = native.load()
    cam = native.Camera(0, 160, 120, 0, 70.0, 70.0, 80.0, 60.0, 0.1, 50.0)
    pairs = (native.Pair * 2)(native.Pair(0, 1, 0, 1, 0, 0, 0.05), native.Pair(1, 2, 1, 2, 0, 0, 0.05))
    cams = (native.Camera * 2)(cam, cam)
    n = ctypes.c_int64(0)
    assert lib.pba_plan_chunks(pairs, 2, cams, 1, 4096, None, None, ctypes.byref(n)) == 0
    assert n.value == 2 * math.ceil(19200 / 4096) and pairs[0].n_chunks == 5
    tab = np.zeros(2 * n.value, np.int32)
    off = np.zeros(3, np.int32)
    assert lib.pba_plan_chunks(pairs, 2, cams, 3, 1024, tab.ctypes.data, off.ctypes.data,
                               ctypes.byref(n)) == 0
    assert off[-1] == n.value == 2 * math.ceil(54 * 40 / 1024)
    # assembly plan: gauge 0, edges (0,1),(1,2),(0,2)
    slot = np.array([-1, 0, 1], np.int32)
    pi = np.array([0, 1, 0], np.int32)
    pj = np.array([1, 2, 2], np.int32)
    n_off = ctypes.c_int32(0)
    assert lib.pba_plan_assembly(slot.ctypes.data, 3, pi.ctypes.data, pj.ctypes.data, 3,
                                 None, None, None, None, None, ctypes.byref(n_off)) == 0
    assert n_off.value == 1
    dp = np.zeros(3, np.int32); di = np.zeros(6, np.int32)
    op = np.zeros(2, np.int32); orc = np.zeros(2, np.int32); oi = np.zeros(3, np.int32)
    assert lib.pba_plan_assembly(slot.ctypes.data, 3, pi.ctypes.data, pj.ctypes.data, 3,
                                 dp.ctypes.data, di.ctypes.data, op.ctypes.data, orc.ctypes.data,
                                 oi.ctypes.data, ctypes.byref(n_off)) == 0
    # slot 0 (pose 1): edge0 side j, edge1 side i ; slot 1 (pose 2): edge1 j, edge2 j
    assert list(dp) == [0, 2, 4]
    assert list(di[:4]) == [(0 << 1) | 1, (1 << 1) | 0, (1 << 1) | 1, (2 << 1) | 1]
    assert list(orc) == [0, 1] and list(oi[:1]) == [(1 << 1) | 0]
    assert lib.pba_plan_chunks(pairs, 2, cams, 0, 1024, None, None, ctypes.byref(n)) == 1
    assert b"stride" in lib.pba_last_error()


def test_new_entry_points_reject_bad_arguments():
    """Argument checks of the round-2 entry points run before any CUDA call
    (so they are exercised here, without a GPU): PBA_ERR_ARG and a message."""
    lib = native.load()
    cam = native.Camera(0, 160, 120, 0, 70.0, 70.0, 80.0, 60.0, 0.1, 50.0)
    assert lib.pba_build_texels_batch(ctypes.byref(cam), -1, None, None, None, None, None, None,
                                      None) == native.PBA_ERR_ARG
    assert b"n_frames" in lib.pba_last_error()
    assert lib.pba_build_texels_batch(ctypes.byref(cam), 0, None, None, None, None, None, None,
                                      None) == native.PBA_OK  # nothing to do
    loop, handle = ctypes.c_void_p(), ctypes.c_uint64()
    assert lib.pba_lm_loop_begin(None, ctypes.byref(loop), ctypes.byref(handle)) == \
        native.PBA_ERR_ARG  # the default stream cannot be captured
    assert lib.pba_lm_decide(None, None, None, None, None, None, 0, None, None, None, 0,
                             None) == native.PBA_ERR_ARG
    buf = ctypes.create_string_buffer(64)
    p = ctypes.addressof(buf)
    assert lib.pba_lm_decide(p, p, p, p, p, p, 0, None, None, None, native.LM_MAX_COPY + 1,
                             None) == native.PBA_ERR_ARG
    assert lib.pba_lm_loop_end(None) == native.PBA_ERR_ARG
    assert lib.pba_lm_loop_launch(None, None) == native.PBA_ERR_ARG
    lib.pba_lm_loop_destroy(None)  # no-op


def test_chunk_plan_whole_row_bands():
    """pba_plan_chunks rounds a pair's chunk to whole 8-row bands when the
    strided grid width is a multiple of 16 and 8 rows fit the requested size
    (K1's 16 x 8 tiled walk, linearize.cu pair_chunk_pixels), else keeps it."""
    lib = native.load()

    def plan(w, h, chunk, stride=1):
        cam = native.Camera(1, w, h, 0, 100.0, 100.0, w / 2, h / 2, 0.1, 50.0)
        pairs = (native.Pair * 1)(native.Pair(0, 1, 0, 1, 0, 0, 0.05))
        cams = (native.Camera * 1)(cam)
        n = ctypes.c_int64(0)
        assert lib.pba_plan_chunks(pairs, 1, cams, stride, chunk, None, None, ctypes.byref(n)) == 0
        tab = np.zeros(2 * n.value, np.int32)
        off = np.zeros(2, np.int32)
        assert lib.pba_plan_chunks(pairs, 1, cams, stride, chunk, tab.ctypes.data,
                                   off.ctypes.data, ctypes.byref(n)) == 0
        assert off[-1] == n.value and (tab[0::2] == 0).all()
        return tab[1::2]

    assert list(plan(1024, 128, 8192)) == [8192 * k for k in range(16)]   # c4: 8 x 1024
    assert list(plan(640, 480, 8192)) == [10240 * k for k in range(30)]   # c3: 16 x 640
    assert list(plan(160, 120, 1024)) == [1024 * k for k in range(19)]    # c1: 8 rows > 1024
    assert list(plan(1000, 64, 8192)) == [8192 * k for k in range(8)]     # width % 16 != 0
    firsts = plan(48, 100, 4096)                                          # 11 bands of 8 rows
    assert list(firsts) == [4224 * k for k in range(2)] and 48 * 100 - firsts[-1] == 576
    assert list(plan(2048, 64, 3072, stride=2)) == [3072 * k for k in range(11)]  # 8 x 1024 > 3072


def test_chunk_size_rule():
    from paper_2303_16878_b200.device import chunk_pixels_for

    # ~32 waves of 444 resident CTAs, 1,024..8,192 pixels; one wave for small problems
    assert chunk_pixels_for(2_519_907_096) == 8192   # c4
    assert chunk_pixels_for(47_316_992) == 3328      # c2
    assert chunk_pixels_for(460_800) == 1024         # c1
    assert chunk_pixels_for(200_000) == 256          # below one wave of 1,024-pixel chunks
    assert chunk_pixels_for(10) == 256


def test_shard_ranges_balanced_and_contiguous():
    from paper_2303_16878_b200.distributed import shard_ranges

    px = [100, 100, 50, 50, 200, 100, 100, 100]
    for world in (1, 2, 3, 4, 8):
        rs = shard_ranges(px, world)
        assert rs[0][0] == 0 and rs[-1][1] == len(px)
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    assert shard_ranges(px, 2) == [(0, 4), (4, 8)]


def test_chunk_orders_are_permutations(monkeypatch):
    from paper_2303_16878_b200.device import order_chunks

    # 3 pairs with 2, 3, 1 chunks of 100 pixels; pairs 0 and 2 share dst frame 5
    tab = np.array([0, 0, 0, 100, 1, 0, 1, 100, 1, 200, 2, 0], np.int32)
    src, dst = [1, 1, 2], [5, 6, 5]
    for order, want in (("pair", [0, 1, 2, 3, 4, 5]), ("dst", [0, 5, 1, 2, 3, 4]),
                        ("src", [0, 2, 1, 3, 4, 5])):
        monkeypatch.setenv("PBA_CHUNK_ORDER", order)
        got = order_chunks(tab.copy(), 6, 100, src, dst).reshape(-1, 2)
        assert [int(np.nonzero((tab.reshape(-1, 2) == r).all(1))[0][0]) for r in got] == want
    # blk with block 2: tiles (src//2, dst//2) = (0,2), (0,3), (1,2) in that order
    monkeypatch.setenv("PBA_CHUNK_ORDER", "blk")
    monkeypatch.setenv("PBA_CHUNK_BLOCK", "2")
    got = order_chunks(tab.copy(), 6, 100, src, dst).reshape(-1, 2)
    idx = [int(np.nonzero((tab.reshape(-1, 2) == r).all(1))[0][0]) for r in got]
    assert idx == [0, 1, 2, 3, 4, 5]
    # default blocks: spherical sources tile by 16, pinhole by 32, models apart
    monkeypatch.setenv("PBA_CHUNK_ORDER", "blk")
    monkeypatch.delenv("PBA_CHUNK_BLOCK")
    got = order_chunks(tab.copy(), 6, 100, src, dst, [1, 0, 1]).reshape(-1, 2)
    idx = [int(np.nonzero((tab.reshape(-1, 2) == r).all(1))[0][0]) for r in got]
    assert idx == [2, 3, 4, 0, 5, 1]  # pair 1 (spherical) first; pinhole pairs 0, 2 interleaved
    # chunk positions are counted inside each pair (pairs may have different chunk sizes)
    monkeypatch.setenv("PBA_CHUNK_ORDER", "dst")
    tab2 = np.array([0, 0, 0, 8192, 1, 0, 1, 10240, 1, 20480, 2, 0], np.int32)
    got = order_chunks(tab2.copy(), 6, 8192, src, dst).reshape(-1, 2)
    idx = [int(np.nonzero((tab2.reshape(-1, 2) == r).all(1))[0][0]) for r in got]
    assert idx == [0, 5, 1, 2, 3, 4]
    monkeypatch.setenv("PBA_CHUNK_ORDER", "bogus")
    with pytest.raises(ValueError):
        order_chunks(tab.copy(), 6, 100, src, dst)


def test_batched_source_points_equal_per_frame():
    """pairgraph._prime_source_points (all frames of a camera at once) gives
    the per-frame _source_points arrays bit for bit."""
    from paper_2303_16878_b200 import pairgraph as G
    from tests import fixtures as F

    for name in ("pinhole_small", "spherical_small"):
        srcs = [lv for p in F.pyramids(F.load(name)) for lv in p.levels]
        for stride in (1, 2, 3):
            one, many = {}, {}
            for s in srcs:
                G._source_points(s, stride, one)
            G._prime_source_points(srcs, stride, many)
            assert one.keys() == many.keys()
            for k, (n, pts, _) in one.items():
                assert many[k][0] == n
                assert (pts is None and many[k][1] is None) or np.array_equal(pts, many[k][1])


def test_bulk_graph_gates_and_transforms_match_scalar_path():
    """The bulk helpers of the device graph build (pairgraph._gated,
    _relative_rows) decide exactly like the per-pair reference path and give
    the same transforms to the last few bits."""
    from paper_2303_16878_b200 import pairgraph as G
    from paper_2303_16878_b200 import scenes as S

    gt = S.room_loop(30)
    poses = S.perturb(gt, 0.3, math.radians(20.0), 5)
    nodes = [P.FrameNode(k, poses[k], None, 0.1 * k) for k in range(30)]
    crit = P.MatchCriteria(max_translation=0.6, max_angle=math.radians(25.0))
    cands = [(a, b) for a in range(30) for b in range(a + 1, 30)]
    want = [ab for ab in cands if G._gates_pass(nodes[ab[0]], nodes[ab[1]], crit)]
    assert 0 < len(want) < len(cands)
    assert G._gated(nodes, cands, crit) == want
    off = P.Pose(np.eye(3), [0.0, 0.0, 0.1])
    sensor = [nd.pose_guess.compose(off) for nd in nodes]
    inv = [sp.inverse() for sp in sensor]
    src = np.array([a for a, b in want] + [b for a, b in want])
    dst = np.array([b for a, b in want] + [a for a, b in want])
    rows = G._relative_rows(sensor, inv, src, dst)
    ref = np.array([G._pose_rows(inv[j].compose(sensor[i])) for i, j in zip(src, dst)])
    assert np.allclose(rows, ref, rtol=0, atol=1e-14)


def test_device_cue_image_depth_without_host_build():
    """DeviceCueImage.depth / depth_valid (used by graph construction) equal
    the host CueImage's clamped depth and mask bit for bit, without building
    the host image."""
    torch = pytest.importorskip("torch")
    from paper_2303_16878_b200.camera import Intrinsics
    from paper_2303_16878_b200.cueimage import CueImage, DeviceCueImage

    cam = Intrinsics(20.0, 20.0, 8.0, 6.0, 16, 12, P.PINHOLE, 0.5, 4.0)
    rng = np.random.default_rng(0)
    d = rng.uniform(0.0, 5.0, (12, 16))
    d[0, 0], d[1, 1], d[2, 2] = np.nan, np.inf, -1.0
    inten = rng.uniform(0, 1, (12, 16))
    nrm = rng.normal(size=(12, 16, 3))
    dev = DeviceCueImage(torch.from_numpy(inten), torch.from_numpy(d), torch.from_numpy(nrm), cam)
    ref = CueImage(inten, d, nrm, cam)
    assert np.array_equal(dev.depth, ref.depth) and dev._host is None
    assert np.array_equal(dev.depth_valid, ref.depth_valid)
    assert np.array_equal(dev.normal_valid, ref.normal_valid)  # builds the host image
    assert np.array_equal(dev.depth, ref.depth)
