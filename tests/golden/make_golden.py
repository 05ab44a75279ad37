"""Generate the golden fixtures of tests/test_oracle_golden.py and
tests/test_gpu_parity.py by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
It imports the read-only reference package from /root/reference/pkg/src and
its test rigs, renders small scenes with the reference renderer and pyramid
builder, and stores inputs (cleaned CueImage channels, derived masks, poses,
edge lists) together with reference outputs:
  - per-pair _EdgeTerm records (solver.py:343-390) at guess and GT poses
  - total_error with and without occlusion suppression (solver.py:655-670)
  - the full LM IterationRecord trace and final poses of solve_hierarchical /
    solve_fusion (solver.py:585-652)
  - the sorted edge list of build_graph (graph.py:123-176)
  - the pyramid index map _footprint_index (cues.py:254-261)
Nothing under tests/golden is read at GPU run time except the .npz files.
"""
import math
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

import numpy as np  # noqa: E402

from photoba.cues import _footprint_index, build_pyramid  # noqa: E402
from photoba.geometry import Pose, boxplus  # noqa: E402
from photoba.graph import FrameNode, MatchCriteria, build_graph  # noqa: E402
from photoba.sensors import PINHOLE, Intrinsics, SensorExtrinsics  # noqa: E402
from photoba.solver import (BAProblem, SolverConfig, _edge_term, _LevelProblem,  # noqa: E402
                            solve_fusion, solve_hierarchical, total_error)
from photoba.synthetic import box_room_scene, render_view  # noqa: E402
from rigs import lidar_cam, loop_trajectory, rgbd_cam, seeded_perturbation  # noqa: E402

OUT = Path(__file__).resolve().parent
IU = np.triu_indices(6)


def cam_row(c):
    return np.array([c.fx, c.fy, c.cx, c.cy, c.width, c.height, 0 if c.model == PINHOLE else 1,
                     c.depth_min, c.depth_max])


def pose_rows(poses):
    return np.stack([np.concatenate([p.rotation.reshape(9), p.translation]) for p in poses])


def term_rows(terms):
    out = np.zeros((len(terms), 92))
    for k, t in enumerate(terms):
        out[k, 90] = t.cost
        out[k, 91] = t.count
        if t.h_ii is not None:
            out[k, 0:21] = t.h_ii[IU]
            out[k, 21:42] = t.h_jj[IU]
            out[k, 42:78] = t.h_ij.reshape(-1)
            out[k, 78:84] = t.b_i
            out[k, 84:90] = t.b_j
    return out


def store_pyramids(d, prefix, pyrs):
    for f, pyr in enumerate(pyrs):
        for l, img in enumerate(pyr.levels):
            d[f"{prefix}I_{f}_{l}"] = img.intensity
            d[f"{prefix}D_{f}_{l}"] = img.depth
            d[f"{prefix}N_{f}_{l}"] = img.normals
            d[f"{prefix}M_{f}_{l}"] = (img.depth_valid.astype(np.uint8)
                                       | (img.normal_valid.astype(np.uint8) << 1)
                                       | ((img.sampleable_intensity & img.sampleable_depth).astype(np.uint8) << 2)
                                       | (img.sampleable_normals.astype(np.uint8) << 3))
            if f == 0:
                d[f"{prefix}G_{f}_{l}"] = np.concatenate(
                    [img.grad_intensity.reshape(-1), img.grad_depth.reshape(-1),
                     img.grad_normals.reshape(-1)])
    d[f"{prefix}cams"] = np.stack([cam_row(img.intrinsics) for img in pyrs[0].levels])
    d[f"{prefix}scales"] = np.array(pyrs[0].scales)


def level_terms(prob, level, poses, cfg, problems=None):
    lp = _LevelProblem(problems or [prob], level, cfg)
    return term_rows([_edge_term(ctx, i, j, poses[i], poses[j], cfg, tol, True)
                      for i, j, ctx, tol in lp.contexts])


def trace_rows(records):
    return np.array([[r.level, r.iteration, r.lam, r.error, r.valid_blocks, r.accepted]
                     for r in records], dtype=float).reshape(-1, 6)


def single_sensor_case(name, cam, n, scales, ext_t, seed, sigma_t, sigma_r):
    gt = loop_trajectory(n).poses
    ext = SensorExtrinsics(Pose(np.eye(3), ext_t))
    room = box_room_scene()
    pyrs = []
    for p in gt:
        r = render_view(room, cam, p.compose(ext.offset))
        pyrs.append(build_pyramid(r.intensity, r.depth, cam, scales))
    rng = np.random.default_rng(seed)
    guess = [gt[0]] + [boxplus(p, seeded_perturbation(rng, sigma_t, sigma_r)) for p in gt[1:]]
    nodes = [FrameNode(k, guess[k], pyrs[k], 0.1 * k) for k in range(n)]
    graph = build_graph(nodes, extrinsics=ext)
    prob = BAProblem(graph, {"sensor0": ext})
    cfg = SolverConfig()
    d = {}
    store_pyramids(d, "", pyrs)
    d["gt"] = pose_rows(gt)
    d["guess"] = pose_rows(guess)
    d["ext"] = np.concatenate([ext.offset.rotation.reshape(9), ext.offset.translation])
    d["edges"] = np.array(graph.edge_pairs(), dtype=np.int64).reshape(-1, 2)
    d["edge_kinds"] = np.array([e.kind == "covisibility" for e in graph.edges])
    for l in range(len(scales)):
        d[f"rec_guess_{l}"] = level_terms(prob, l, guess, cfg)
        d[f"rec_gt_{l}"] = level_terms(prob, l, gt, cfg)
        d[f"te_{l}"] = np.array([*total_error(prob, guess, l, cfg),
                                 *total_error(prob, guess, l, cfg, suppress_occlusions=False)])
    res = solve_hierarchical(prob, cfg)
    d["trace"] = trace_rows(res.records)
    d["final"] = pose_rows(res.poses)
    np.savez_compressed(OUT / f"{name}.npz", **d)
    print(name, len(graph.edges), "edges;", len(res.records), "LM records;",
          (OUT / f"{name}.npz").stat().st_size, "bytes")


def fusion_case():
    from rigs import LIDAR_EXTRINSICS, RGBD_EXTRINSICS
    rgbd = Intrinsics(40.0, 40.0, 32.0, 24.0, 64, 48, PINHOLE, 0.1, 50.0)
    lidar = Intrinsics(128 / (2 * math.pi), 32 / (math.pi / 2), 64.0, 16.0, 128, 32, "spherical",
                       0.2, 80.0)
    gt = Pose(np.eye(3), [-0.4, -0.2, -0.6])
    rng = np.random.default_rng(4242)
    bad = boxplus(gt, seeded_perturbation(rng, 0.05, 0.03))
    room = box_room_scene()
    d = {}
    probs = []
    for tag, cam, ext in (("r_", rgbd, RGBD_EXTRINSICS), ("l_", lidar, LIDAR_EXTRINSICS)):
        r = render_view(room, cam, gt.compose(ext.offset))
        pyr = build_pyramid(r.intensity, r.depth, cam, (0.5, 1.0))
        store_pyramids(d, tag, [pyr])
        sid = "rgbd" if tag == "r_" else "lidar"
        nodes = [FrameNode(0, gt, pyr, 0.0, sid), FrameNode(1, bad, pyr, 0.1, sid)]
        from photoba.graph import Edge, MatchGraph
        probs.append(BAProblem(MatchGraph(nodes, [Edge(0, 1, "covisibility")]), {sid: ext}))
        d[tag + "ext"] = np.concatenate([ext.offset.rotation.reshape(9), ext.offset.translation])
    d["gt"] = pose_rows([gt, gt])
    d["guess"] = pose_rows([gt, bad])
    cfg = SolverConfig()
    for l in range(2):
        d[f"rec_guess_{l}"] = level_terms(None, l, [gt, bad], cfg, probs)
    res = solve_fusion(probs[0], probs[1], "coupled", cfg)
    d["trace"] = trace_rows(res.records)
    d["final"] = pose_rows(res.poses)
    res2 = solve_fusion(probs[1], probs[0], "consecutive", cfg)
    d["trace_consecutive"] = trace_rows(res2.records)
    d["final_consecutive"] = pose_rows(res2.poses)
    np.savez_compressed(OUT / "fusion_small.npz", **d)
    print("fusion_small", len(res.records), (OUT / "fusion_small.npz").stat().st_size, "bytes")


def footprint_case():
    d = {}
    for k, (h, w, s) in enumerate([(11, 15, 1 / 3), (460, 740, 0.125), (128, 1024, 0.25),
                                   (96, 128, 0.5), (57, 93, 0.7), (64, 1024, 1.0)]):
        idx, keep, oh, ow = _footprint_index(h, w, s)
        d[f"fp_{k}"] = np.array([h, w, s, oh, ow])
        # the map is separable: row index of column 0 and column index of row 0
        d[f"fp_rows_{k}"] = np.where(keep[:, 0], idx[:, 0] // max(ow, 1), -1).astype(np.int32)
        d[f"fp_cols_{k}"] = np.where(keep[0, :], idx[0, :] % max(ow, 1), -1).astype(np.int32)
        d[f"fp_sum_{k}"] = np.array([int(idx[keep].sum()), int(keep.sum())])
    np.savez_compressed(OUT / "footprint.npz", **d)


def pyramid_case():
    """Raw renders + the reference's estimate_normals / build_pyramid outputs
    (cues.py:187-375) for a pinhole and a spherical sensor."""
    from photoba.cues import estimate_normals
    d = {}
    room = box_room_scene()
    cams = [("p", rgbd_cam(), Pose(np.eye(3), [-0.4, 0.2, -0.5]), (0.25, 0.5, 1.0)),
            ("s", lidar_cam(128, 32), Pose(np.eye(3), [0.3, -0.2, 0.1]), (0.25, 0.5, 1.0))]
    for tag, cam, pose, scales in cams:
        r = render_view(room, cam, pose)
        depth = r.depth.copy()
        rng = np.random.default_rng(5)
        depth[rng.random(depth.shape) < 0.02] = 0.0  # holes
        depth[3, 5] = np.nan
        d[f"{tag}_cam"] = cam_row(cam)
        d[f"{tag}_I"] = r.intensity
        d[f"{tag}_D"] = depth
        d[f"{tag}_normals"] = estimate_normals(depth, cam)
        pyr = build_pyramid(r.intensity, depth, cam, scales)
        d[f"{tag}_scales"] = np.array(scales)
        for l, img in enumerate(pyr.levels):
            d[f"{tag}_I_{l}"] = img.intensity
            d[f"{tag}_D_{l}"] = img.depth
            d[f"{tag}_N_{l}"] = img.normals
            d[f"{tag}_cam_{l}"] = cam_row(img.intrinsics)
    np.savez_compressed(OUT / "pyramid.npz", **d)
    print("pyramid", (OUT / "pyramid.npz").stat().st_size, "bytes")


def behaviour_case():
    """Raw renders (intensity, depth) and seeded perturbations for the
    reference's behavioural solver tests (test_solver.py:374-563), so the
    same scenarios run on the GPU path (pyramids are rebuilt with the
    package's bit-exact build_pyramid)."""
    from rigs import LIDAR_EXTRINSICS, RGBD_EXTRINSICS

    d = {}
    cam_r, cam_l = rgbd_cam(), lidar_cam()
    d["cam_rgbd"], d["cam_lidar"] = cam_row(cam_r), cam_row(cam_l)
    room = box_room_scene()

    def view(tag, cam, pose, ext=None):
        off = ext.offset if ext is not None else Pose.identity()
        r = render_view(room, cam, pose.compose(off))
        d[f"{tag}_I"], d[f"{tag}_D"] = r.intensity, r.depth

    view("zero", cam_r, Pose.identity())
    view("selfalign", cam_r, Pose(np.eye(3), [-0.5, -0.3, -0.8]))
    view("optimal", cam_r, Pose(np.eye(3), [-0.4, 0.2, -0.5]))
    gt_f = Pose(np.eye(3), [-0.4, -0.2, -0.6])
    view("fusion_rgbd", cam_r, gt_f, RGBD_EXTRINSICS)
    view("fusion_lidar", cam_l, gt_f, LIDAR_EXTRINSICS)
    loop = loop_trajectory(5)
    for k, p in enumerate(loop.poses):
        view(f"loop{k}", cam_r, p)
    d["loop_gt"] = pose_rows(loop.poses)
    gt_s = Pose(np.eye(3), [-0.5, -0.3, -0.8])
    d["selfalign_bad"] = pose_rows([boxplus(gt_s, seeded_perturbation(np.random.default_rng(47), 0.1, 0.0))])
    d["monotone_bad"] = pose_rows([boxplus(gt_s, seeded_perturbation(np.random.default_rng(48), 0.12, 0.08))])
    d["coupled_bad"] = pose_rows([boxplus(gt_f, seeded_perturbation(np.random.default_rng(4242), 0.25, 0.3))])
    rng = np.random.default_rng(51)
    d["loop_guess"] = pose_rows([loop.poses[0]] + [
        boxplus(p, seeded_perturbation(rng, 0.04, math.radians(1.5))) for p in loop.poses[1:]])
    np.savez_compressed(OUT / "behaviour.npz", **d)
    print("behaviour", (OUT / "behaviour.npz").stat().st_size, "bytes")


def acceptance_case():
    """Inputs of the reference's acceptance criteria (test_acceptance.py:60-255):
    the 10-pose recovery case (loop_trajectory(10), perturb_trajectory seed 11),
    the hierarchical-benefit case (seed 3) and the 5x5 fusion-ordering grid
    (seed 42); renders are raw intensity/depth."""
    from photoba.synthetic import perturb_trajectory

    d = {}
    cam = rgbd_cam()
    room = box_room_scene()
    gt = loop_trajectory(10)
    for k, p in enumerate(gt.poses):
        r = render_view(room, cam, p)
        d[f"loop10_{k}_I"], d[f"loop10_{k}_D"] = r.intensity, r.depth
    d["loop10_gt"] = pose_rows(gt.poses)
    d["loop10_stamps"] = gt.timestamps
    d["loop10_guess"] = pose_rows(perturb_trajectory(gt, 0.05, math.radians(2.0), seed=11).poses)
    rng = np.random.default_rng(3)
    d["benefit_bad2"] = pose_rows([boxplus(gt.poses[2], seeded_perturbation(rng, 0.22, 0.22))])
    gt_f = Pose(np.eye(3), [-0.4, -0.2, -0.6])
    rng = np.random.default_rng(42)
    bad = []
    for r_mag in np.linspace(0.0, 0.3, 5):
        for t_mag in np.linspace(0.0, 0.3, 5):
            bad.append(boxplus(gt_f, seeded_perturbation(rng, t_mag, r_mag)))
    d["fusion_grid_bad"] = pose_rows(bad)
    np.savez_compressed(OUT / "acceptance.npz", **d)
    print("acceptance", (OUT / "acceptance.npz").stat().st_size, "bytes")


def evaluation_case():
    """associate / horn_align / evaluate_ate (evaluation.py:48-122) on
    seeded trajectories: timestamp jitter, dropped poses, a rigid offset and
    pose noise."""
    from photoba.evaluation import Trajectory, associate, evaluate_ate

    rng = np.random.default_rng(11)
    d = {}
    for case in range(4):
        n = 40 + 10 * case
        ts = np.cumsum(rng.uniform(0.05, 0.15, n))
        ref = [boxplus(Pose(np.eye(3), rng.normal(0, 2.0, 3)), seeded_perturbation(rng, 0.0, 0.5))
               for _ in range(n)]
        g = boxplus(Pose(np.eye(3), [1.0, -2.0, 0.5]), seeded_perturbation(rng, 0.0, 0.7))
        keep = np.sort(rng.choice(n, n - 5, replace=False))
        est_ts = ts[keep] + rng.uniform(-0.01, 0.01, keep.size)
        order = np.argsort(est_ts)
        est = [g.compose(boxplus(ref[k], seeded_perturbation(rng, 0.02, 0.01))) for k in keep[order]]
        tr_ref = Trajectory(ts, ref)
        tr_est = Trajectory(est_ts[order], est)
        pairs = associate(tr_est, tr_ref, 0.02)
        rep = evaluate_ate(tr_est, tr_ref, 0.02)
        d[f"ref_ts_{case}"] = ts
        d[f"ref_{case}"] = pose_rows(ref)
        d[f"est_ts_{case}"] = tr_est.timestamps
        d[f"est_{case}"] = pose_rows(est)
        d[f"pairs_{case}"] = np.array(pairs, dtype=np.int64)
        d[f"report_{case}"] = np.array([rep.rmse, rep.rotation_rmse, rep.matches])
        d[f"align_{case}"] = pose_rows([rep.alignment])[0]
    np.savez_compressed(OUT / "evaluation.npz", **d)
    print("evaluation", (OUT / "evaluation.npz").stat().st_size, "bytes")


def dataset_case():
    """A two-sensor dataset directory written by the reference's
    generate_synthetic (synthetic.py:257-310), stored file by file, plus the
    reference load_dataset output (dataset_io.py:305-342)."""
    import tempfile

    from photoba.dataset_io import load_dataset
    from photoba.evaluation import Trajectory
    from photoba.synthetic import SyntheticSensor, generate_synthetic

    traj = Trajectory(np.arange(3, dtype=float) * 0.1 + 0.05,
                      [Pose(np.eye(3), [0.1 * k, 0.05 * k, -0.5]) for k in range(3)])
    sensors = [SyntheticSensor("cam0", rgbd_cam(), SensorExtrinsics.identity(), 0.001),
               SyntheticSensor("lidar0", lidar_cam(128, 32),
                               SensorExtrinsics(Pose(np.eye(3), [0.0, 0.0, 0.1])), 0.002)]
    d = {}
    with tempfile.TemporaryDirectory() as tmp:
        ds = generate_synthetic(box_room_scene(), traj, sensors, Path(tmp) / "ds",
                                pyramid_scales=(0.25, 0.5, 1.0))
        files = sorted(p for p in ds.rglob("*") if p.is_file())
        d["files"] = np.array([str(p.relative_to(ds)) for p in files])
        for k, p in enumerate(files):
            d[f"file_{k}"] = np.frombuffer(p.read_bytes(), dtype=np.uint8)
        _, guess, frames = load_dataset(ds)
        d["guess"] = pose_rows(guess.poses)
        d["stamps"] = guess.timestamps
        for sid, nodes in frames.items():
            for f, node in enumerate(nodes):
                for l, img in enumerate(node.pyramid.levels):
                    if f > 0 and l < len(node.pyramid.levels) - 1:
                        continue  # all levels of frame 0, the finest of the others
                    d[f"{sid}_I_{f}_{l}"] = img.intensity
                    d[f"{sid}_D_{f}_{l}"] = img.depth
                    d[f"{sid}_N_{f}_{l}"] = img.normals
    np.savez_compressed(OUT / "dataset.npz", **d)
    print("dataset", len(d["files"]), "files", (OUT / "dataset.npz").stat().st_size, "bytes")


def utility_case():
    """The reference's public utilities beside the solver: reproject
    (solver.py:154-176) and sample (cues.py:412-430), on a rendered cue image
    with holes and random continuous pixels (inside, on the border, outside)."""
    from photoba.cues import CueImage, sample
    from photoba.geometry import PerturbationVector, exp
    from photoba.solver import reproject

    rng = np.random.default_rng(77)
    d = {}
    pin = rgbd_cam()
    sph = lidar_cam(256, 32)
    for tag, cam in (("pin", pin), ("sph", sph)):
        d[f"{tag}_cam"] = cam_row(cam)
        m = 400
        uv = np.stack([rng.uniform(0, cam.width - 1, m), rng.uniform(0, cam.height - 1, m)], -1)
        depth = rng.uniform(cam.depth_min, min(cam.depth_max, 8.0), m)
        xi = exp(PerturbationVector(rng.normal(0, 0.3, 3), rng.normal(0, 0.1, 3)))
        xj = exp(PerturbationVector(rng.normal(0, 0.3, 3), rng.normal(0, 0.1, 3)))
        off = exp(PerturbationVector(rng.normal(0, 0.05, 3), rng.normal(0, 0.05, 3)))
        uv_dst, p_bar, valid = reproject(uv, depth, xi, xj, SensorExtrinsics(off), cam, cam)
        d[f"{tag}_uv"], d[f"{tag}_depth"] = uv, depth
        d[f"{tag}_xi"], d[f"{tag}_xj"], d[f"{tag}_off"] = pose_rows([xi]), pose_rows([xj]), pose_rows([off])
        d[f"{tag}_uv_dst"], d[f"{tag}_p_bar"], d[f"{tag}_valid"] = uv_dst, p_bar, valid
    # sample: one rendered RGB-D view with estimated normals and punched holes
    r = render_view(box_room_scene(), pin, Pose(np.eye(3), [-0.4, 0.2, -0.5]))
    pyr = build_pyramid(r.intensity, r.depth, pin, (1.0,))
    img0 = pyr.levels[0]
    depth = img0.depth.copy()
    depth[rng.random(depth.shape) < 0.03] = 0.0
    img = CueImage(img0.intensity, depth, img0.normals, pin)
    d["img_I"], d["img_D"], d["img_N"] = img.intensity, img.depth, img.normals
    m = 600
    uv = np.stack([rng.uniform(-2, pin.width + 1, m), rng.uniform(-2, pin.height + 1, m)], -1)
    uv[:20] = np.floor(uv[:20])                              # exact pixel centres
    uv[20:30, 0] = pin.width - 1.0                           # right border (wx = 1)
    uv[30:40, 1] = pin.height - 1.0                          # bottom border
    d["sample_uv"] = uv
    for ch in ("intensity", "depth", "normals"):
        v, g, ok = sample(img, uv, ch)
        d[f"sample_{ch}_v"], d[f"sample_{ch}_g"], d[f"sample_{ch}_ok"] = v, g, ok
        v1, g1, ok1 = sample(img, uv[5], ch)                  # single-point form
        d[f"sample1_{ch}_v"], d[f"sample1_{ch}_g"], d[f"sample1_{ch}_ok"] = v1, g1, ok1
    np.savez_compressed(OUT / "utility.npz", **d)
    print("utility", (OUT / "utility.npz").stat().st_size, "bytes")


if __name__ == "__main__":
    cases = set(sys.argv[1:])  # empty: regenerate everything

    def want(name):
        return not cases or name in cases

    if want("pinhole_small"):
        pin = Intrinsics(40.0, 40.0, 32.0, 24.0, 64, 48, PINHOLE, 0.1, 50.0)
        single_sensor_case("pinhole_small", pin, 4, (1.0,), [0.0, 0.0, 0.1], 51, 0.04,
                           math.radians(1.5))
    if want("spherical_small"):
        sph = Intrinsics(128 / (2 * math.pi), 24 / (math.pi / 2), 64.0, 12.0, 128, 24,
                         "spherical", 0.2, 80.0)
        single_sensor_case("spherical_small", sph, 4, (0.5, 1.0), [0.0, 0.0, -0.05], 52, 0.04,
                           math.radians(1.5))
    for name, fn in (("fusion", fusion_case), ("footprint", footprint_case),
                     ("pyramid", pyramid_case), ("dataset", dataset_case),
                     ("evaluation", evaluation_case), ("behaviour", behaviour_case),
                     ("acceptance", acceptance_case), ("utility", utility_case)):
        if want(name):
            fn()
