"""Pin the C oracle (oracle/pba_oracle.c + oracle/oracle.py) against vectors
produced by the reference implementation itself (tests/golden/*.npz).
CPU only."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from tests import fixtures as F

CASES = ["pinhole_small", "spherical_small"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_derivation_matches_reference_cueimage(name):
    d = F.load(name)
    cams = [F.cam_from_row(r) for r in d["cams"]]
    f = 0
    while f"I_{f}_0" in d:
        for l, cam in enumerate(cams):
            img = O.derive_image(d[f"I_{f}_{l}"], d[f"D_{f}_{l}"], d[f"N_{f}_{l}"], cam)
            bits = (img.depth_valid | (img.normal_valid << 1) | (img.sampleable_core << 2)
                    | (img.sampleable_normals << 3))
            assert np.array_equal(bits, d[f"M_{f}_{l}"])
            assert np.array_equal(img.depth, d[f"D_{f}_{l}"])
            assert np.array_equal(img.normals, d[f"N_{f}_{l}"])
            if f == 0:
                g = np.concatenate([img.grad_intensity.reshape(-1), img.grad_depth.reshape(-1),
                                    img.grad_normals.reshape(-1)])
                assert np.array_equal(g, d[f"G_{f}_{l}"])
        f += 1


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("which", ["guess", "gt"])
def test_oracle_edge_terms_match_reference(name, which):
    d = F.load(name)
    prob, _ = F.single_problem(d)
    cfg = O_cfg()
    pose_arr = d[which]
    for l in range(len(d["scales"])):
        lp = O.OracleLevel([prob], l, cfg)
        recs = lp.records(pose_arr)
        F.compare_records(recs, d[f"rec_{which}_{l}"], h_tol=1e-11, b_tol=1e-8, cost_tol=1e-10)


@pytest.mark.parametrize("name", CASES)
def test_oracle_total_error_matches_reference(name):
    d = F.load(name)
    prob, _ = F.single_problem(d)
    cfg = O_cfg()
    guess = F.poses(d["guess"])
    for l in range(len(d["scales"])):
        c1, n1, c2, n2 = d[f"te_{l}"]
        cost, count = O.total_error(prob, guess, l, cfg)
        assert count == int(n1) and abs(cost - c1) <= 1e-12 * c1
        cost, count = O.total_error(prob, guess, l, cfg, suppress_occlusions=False)
        assert count == int(n2) and abs(cost - c2) <= 1e-12 * c2


@pytest.mark.parametrize("name", CASES)
def test_oracle_lm_trace_matches_reference(name):
    d = F.load(name)
    prob, _ = F.single_problem(d)
    final, records = O.hierarchical([prob], O_cfg())
    trace = d["trace"]
    assert len(records) == len(trace)
    for r, t in zip(records, trace):
        assert (r.level, r.iteration, int(r.accepted), r.valid_blocks) == (
            int(t[0]), int(t[1]), int(t[5]), int(t[4]))
        assert r.lam == t[2]
        assert abs(r.error - t[3]) <= 1e-9 * abs(t[3])
    assert np.max(np.abs(final - d["final"])) < 1e-9


def test_oracle_fusion_coupled_matches_reference():
    d = F.load("fusion_small")
    probs = F.fusion_problems(d)
    for l in range(2):
        lp = O.OracleLevel(probs, l, O_cfg())
        F.compare_records(lp.records(d["guess"]), d[f"rec_guess_{l}"], 1e-11, 1e-8, 1e-10)
    final, records = O.hierarchical(probs, O_cfg())
    assert [(r.level, r.iteration, r.accepted) for r in records] == [
        (int(t[0]), int(t[1]), bool(t[5])) for t in d["trace"]]
    assert np.max(np.abs(final - d["final"])) < 1e-9


def O_cfg():
    from paper_2303_16878_b200 import SolverConfig

    return SolverConfig()
