"""Load the golden fixtures (tests/golden/*.npz, produced by the reference
via tests/golden/make_golden.py) into the package's drop-in types."""
from __future__ import annotations

from pathlib import Path

import numpy as np

import paper_2303_16878_b200 as P

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def cam_from_row(r) -> P.Intrinsics:
    return P.Intrinsics(float(r[0]), float(r[1]), float(r[2]), float(r[3]), int(r[4]), int(r[5]),
                        P.PINHOLE if int(r[6]) == 0 else P.SPHERICAL, float(r[7]), float(r[8]))


def pyramids(d: dict, prefix: str = "") -> list:
    cams = [cam_from_row(r) for r in d[prefix + "cams"]]
    scales = tuple(float(s) for s in d[prefix + "scales"])
    out, f = [], 0
    while f"{prefix}I_{f}_0" in d:
        levels = tuple(P.CueImage(d[f"{prefix}I_{f}_{l}"], d[f"{prefix}D_{f}_{l}"],
                                  d[f"{prefix}N_{f}_{l}"], cams[l]) for l in range(len(cams)))
        out.append(P.CuePyramid(levels, scales))
        f += 1
    return out


def poses(rows) -> list:
    return [P.Pose.from_row(r) for r in rows]


def single_problem(d: dict, use_guess: bool = True):
    pyrs = pyramids(d)
    guess = poses(d["guess"])
    nodes = [P.FrameNode(k, guess[k], pyrs[k], 0.1 * k) for k in range(len(pyrs))]
    kinds = d["edge_kinds"]
    edges = [P.Edge(int(i), int(j), P.COVISIBILITY if kinds[k] else P.ODOMETRY)
             for k, (i, j) in enumerate(d["edges"])]
    ext = P.SensorExtrinsics(P.Pose.from_row(d["ext"]))
    return P.BAProblem(P.MatchGraph(nodes, edges), {"sensor0": ext}), ext


def fusion_problems(d: dict):
    probs = []
    guess = poses(d["guess"])
    for tag, sid in (("r_", "rgbd"), ("l_", "lidar")):
        pyr = pyramids(d, tag)[0]
        nodes = [P.FrameNode(0, guess[0], pyr, 0.0, sid), P.FrameNode(1, guess[1], pyr, 0.1, sid)]
        ext = P.SensorExtrinsics(P.Pose.from_row(d[tag + "ext"]))
        probs.append(P.BAProblem(P.MatchGraph(nodes, [P.Edge(0, 1, P.COVISIBILITY)]), {sid: ext}))
    return probs


def mask_bits(img) -> np.ndarray:
    return (img.depth_valid.astype(np.uint8) | (img.normal_valid.astype(np.uint8) << 1)
            | ((img.sampleable_intensity & img.sampleable_depth).astype(np.uint8) << 2)
            | (img.sampleable_normals.astype(np.uint8) << 3))


def rel(a, b) -> float:
    a, b = np.asarray(a, float), np.asarray(b, float)
    den = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / den) if den > 0 else float(np.max(np.abs(a - b)))


def compare_records(got, ref, h_tol=1e-5, b_tol=1e-5, cost_tol=1e-6):
    """SURVEY.md §8(c) parity metrics per pair: counts equal, H/b max|Δ|/max|ref|,
    cost relative.  b -> 0 at convergence (and is pure rounding noise at an
    exact self-alignment), so b's error is also accepted relative to the
    Cauchy-Schwarz scale of its terms, sqrt(max diag H * cost) — the
    |Δb| / Σ|JᵀWe| normalisation of SURVEY.md §8(c)."""
    got, ref = np.asarray(got), np.asarray(ref)
    assert got.shape == ref.shape
    assert np.array_equal(got[:, 91], ref[:, 91]), (got[:, 91], ref[:, 91])
    for k in range(ref.shape[0]):
        if ref[k, 91] == 0:
            assert np.all(got[k, :91] == 0.0)
            continue
        for lo, hi, tol in ((0, 21, h_tol), (21, 42, h_tol), (42, 78, h_tol)):
            assert rel(got[k, lo:hi], ref[k, lo:hi]) <= tol, (k, lo, rel(got[k, lo:hi], ref[k, lo:hi]))
        diag = [0, 6, 11, 15, 18, 20]
        hmax = max(np.max(np.abs(ref[k, diag])), np.max(np.abs(ref[k, [21 + d for d in diag]])))
        scale = np.sqrt(hmax * max(ref[k, 90], 0.0))
        for lo, hi in ((78, 84), (84, 90)):
            err = np.max(np.abs(got[k, lo:hi] - ref[k, lo:hi]))
            # absolute floor: the reference's own self-alignment bound |b| < 1e-10
            # (pkg/tests/test_solver.py:414-420) — b is rounding noise there
            assert err <= max(b_tol * max(np.max(np.abs(ref[k, lo:hi])), 1e-6 * scale), 1e-10), (
                k, lo, err)
        # cost: relative, or inside the reference's noise floor of 1e-18 per
        # valid block (solver.py:490-492) — e.g. an exact self-alignment
        assert abs(got[k, 90] - ref[k, 90]) <= cost_tol * abs(ref[k, 90]) + 1e-18 * ref[k, 91], (
            k, got[k, 90], ref[k, 90])
