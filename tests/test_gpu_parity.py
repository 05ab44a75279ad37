"""GPU parity: the sm_100a path (through the C ABI) against the oracle and
the reference's own golden vectors.  Tolerances are SURVEY.md §8(c):
per-pair H/b max|Δ|/max|ref| <= 1e-5, cost <= 1e-6 relative, counts equal,
LM trace equal in (level, iteration, accepted, count, lambda), final poses
<= 1e-5 rad / 1e-5 m."""
import math

import numpy as np
import pytest

import paper_2303_16878_b200 as P
from oracle import oracle as O
from tests import fixtures as F

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CASES = ["pinhole_small", "spherical_small"]


def _store():
    from paper_2303_16878_b200.device import FrameStore

    return FrameStore(torch.device("cuda", 0))


def _level(problems, level, cfg=None, **kw):
    from paper_2303_16878_b200.device import DeviceLevel

    return DeviceLevel(problems, level, cfg or P.SolverConfig(), _store(), **kw)


def _rows(arr):
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).cuda()


def _pose_err(a_rows, b_rows):
    worst_r = worst_t = 0.0
    for a, b in zip(a_rows, b_rows):
        Ra, Rb = a[:9].reshape(3, 3), b[:9].reshape(3, 3)
        worst_r = max(worst_r, P.rotation_angle(Rb.T @ Ra))
        worst_t = max(worst_t, float(np.linalg.norm(a[9:] - b[9:])))
    return worst_r, worst_t


@pytest.mark.parametrize("name", CASES)
def test_device_texels_bit_exact_masks_and_gradients(name):
    d = F.load(name)
    store = _store()
    for f, pyr in enumerate(F.pyramids(d)):
        for l, img in enumerate(pyr.levels):
            tex, mask, _, _ = store.frame(img)
            torch.cuda.synchronize()
            m = mask.cpu().numpy().reshape(img.shape)
            assert np.array_equal(m, d[f"M_{f}_{l}"])
            # eight planes of (h, w) 16-byte pairs, see include/pba.h
            t = tex.cpu().numpy().view(np.float64).reshape(8, img.shape[0], img.shape[1], 2)
            assert np.array_equal(t[0, ..., 0], img.intensity)
            assert np.array_equal(t[0, ..., 1], img.depth)
            assert np.array_equal(np.stack([t[1, ..., 0], t[1, ..., 1], t[2, ..., 0]], -1),
                                  img.normals)
            words = t[2, ..., 1].view(np.uint64) & 0xFFFFFFFF
            assert np.array_equal(words, m.astype(np.uint64))
            if f == 0:
                g = np.concatenate([t[3].reshape(-1), t[4].reshape(-1),
                                    np.stack([t[5], t[6], t[7]], axis=2).reshape(-1)])
                assert np.array_equal(g, d[f"G_{f}_{l}"])


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("which", ["guess", "gt"])
def test_linearize_matches_reference_records(name, which):
    d = F.load(name)
    prob, _ = F.single_problem(d)
    for l in range(len(d["scales"])):
        lv = _level([prob], l)
        recs = lv.linearize(_rows(d[which])).cpu().numpy()
        F.compare_records(recs, d[f"rec_{which}_{l}"])
        # and against the oracle on the same inputs
        ol = O.OracleLevel([prob], l, P.SolverConfig())
        F.compare_records(recs, ol.records(d[which]))


@pytest.mark.parametrize("name", CASES)
def test_total_error_matches_reference(name):
    d = F.load(name)
    prob, _ = F.single_problem(d)
    guess = F.poses(d["guess"])
    for l in range(len(d["scales"])):
        c1, n1, c2, n2 = d[f"te_{l}"]
        cost, count = P.total_error(prob, guess, l)
        assert count == int(n1) and abs(cost - c1) <= 1e-6 * c1
        cost, count = P.total_error(prob, guess, l, suppress_occlusions=False)
        assert count == int(n2) and abs(cost - c2) <= 1e-6 * c2


def _check_trace(records, trace, err_tol=1e-6):
    """Record trace equal in (level, iteration, accepted, count, lambda); cost
    within 1e-6 relative, or both inside the reference's own floating-point
    noise floor of 1e-18 per valid block (solver.py:490-492)."""
    assert len(records) == len(trace), (len(records), len(trace))
    for r, t in zip(records, trace):
        assert (r.level, r.iteration, int(r.accepted), r.valid_blocks) == (
            int(t[0]), int(t[1]), int(t[5]), int(t[4]))
        assert r.lam == t[2]
        assert abs(r.error - t[3]) <= err_tol * abs(t[3]) + 1e-18 * max(1, t[4])


@pytest.mark.parametrize("name", CASES)
def test_solve_hierarchical_matches_reference_trace(name):
    d = F.load(name)
    prob, _ = F.single_problem(d)
    res = P.solve_hierarchical(prob)
    _check_trace(res.records, d["trace"])
    final = np.stack([p.as_row() for p in res.poses])
    er, et = _pose_err(final, d["final"])
    assert er <= 1e-5 and et <= 1e-5


def test_fusion_matches_reference():
    d = F.load("fusion_small")
    probs = F.fusion_problems(d)
    for l in range(2):
        lv = _level(probs, l)
        F.compare_records(lv.linearize(_rows(d["guess"])).cpu().numpy(), d[f"rec_guess_{l}"])
    res = P.solve_fusion(probs[0], probs[1], "coupled")
    _check_trace(res.records, d["trace"])
    er, et = _pose_err(np.stack([p.as_row() for p in res.poses]), d["final"])
    assert er <= 1e-5 and et <= 1e-5
    res2 = P.solve_fusion(probs[1], probs[0], "consecutive")
    _check_trace(res2.records, d["trace_consecutive"])
    er, et = _pose_err(np.stack([p.as_row() for p in res2.poses]), d["final_consecutive"])
    assert er <= 1e-5 and et <= 1e-5


# ---------------------------------------------------------------------------
# larger synthetic problems against the oracle (BASELINE config 1 shape etc.)
# ---------------------------------------------------------------------------
def _room_problem(n=10, cam=None, scales=(1.0,), seed=11):
    from paper_2303_16878_b200 import scenes as S

    cam = cam or S.rgbd_160()
    gt = S.room_loop(n)
    pyrs = S.host_pyramids(S.BoxScene(), cam, gt, P.Pose.identity(), scales)
    guess = S.perturb(gt, 0.05, math.radians(2.0), seed)
    nodes = [P.FrameNode(k, guess[k], pyrs[k], 0.1 * k) for k in range(n)]
    return P.BAProblem(P.build_graph(nodes)), gt, guess


def test_config1_linearize_matches_oracle():
    prob, gt, guess = _room_problem()
    assert len(prob.graph.edges) == 24
    rows, _ = P.se3.pose_rows(guess)
    lv = _level([prob], 0)
    got = lv.linearize(_rows(rows)).cpu().numpy()
    ref = O.OracleLevel([prob], 0, P.SolverConfig()).records(rows)
    F.compare_records(got, ref)
    assert int(got[:, 91].sum()) > 0.8 * 24 * 160 * 120 * 0.5


def test_config1_lm_trace_matches_oracle():
    prob, gt, guess = _room_problem()
    res = P.solve_hierarchical(prob)
    final_o, recs_o = O.hierarchical([prob], P.SolverConfig())
    assert [(r.level, r.iteration, r.accepted, r.valid_blocks) for r in res.records] == [
        (r.level, r.iteration, r.accepted, r.valid_blocks) for r in recs_o]
    assert [r.lam for r in res.records] == [r.lam for r in recs_o]
    for a, b in zip(res.records, recs_o):
        assert abs(a.error - b.error) <= 1e-6 * b.error
    er, et = _pose_err(np.stack([p.as_row() for p in res.poses]), final_o)
    assert er <= 1e-5 and et <= 1e-5


def test_spherical_corridor_linearize_matches_oracle():
    from paper_2303_16878_b200 import scenes as S

    cam = S.hdl64(512, 64)
    gt = S.corridor_trajectory(6, 0.5)
    ext = P.Pose.identity()
    pyrs = S.host_pyramids(S.corridor_scene(23.0), cam, gt, ext, (0.25, 0.5, 1.0))
    guess = S.perturb(gt, 0.05, math.radians(2.0), 11)
    nodes = [P.FrameNode(k, guess[k], pyrs[k], 0.1 * k) for k in range(len(gt))]
    prob = P.BAProblem(P.build_graph(nodes))
    rows, _ = P.se3.pose_rows(guess)
    for l in range(3):
        got = _level([prob], l).linearize(_rows(rows)).cpu().numpy()
        ref = O.OracleLevel([prob], l, P.SolverConfig()).records(rows)
        F.compare_records(got, ref)


def test_pixel_stride_and_cost_only_path():
    prob, gt, guess = _room_problem(n=5, scales=(0.5, 1.0))
    rows, _ = P.se3.pose_rows(guess)
    cfg = P.SolverConfig(pixel_stride=3)
    got = _level([prob], 1, cfg).linearize(_rows(rows)).cpu().numpy()
    ref = O.OracleLevel([prob], 1, cfg).records(rows)
    F.compare_records(got, ref)
    got = _level([prob], 1, cfg).linearize(_rows(rows), want_jacobians=False).cpu().numpy()
    ref = O.OracleLevel([prob], 1, cfg).records(rows, want_jacobians=False)
    assert np.array_equal(got[:, 91], ref[:, 91])
    assert np.allclose(got[:, 90], ref[:, 90], rtol=1e-9)
    assert np.all(got[:, :90] == 0.0)


def test_deterministic_and_shard_independent():
    prob, gt, guess = _room_problem()
    rows, _ = P.se3.pose_rows(guess)
    full = _level([prob], 0).linearize(_rows(rows)).cpu().numpy()
    again = _level([prob], 0).linearize(_rows(rows)).cpu().numpy()
    assert np.array_equal(full, again)
    parts = [_level([prob], 0, pair_range=r, assemble=False).linearize(_rows(rows)).cpu().numpy()
             for r in [(0, 7), (7, 15), (15, 24)]]
    assert np.array_equal(np.concatenate(parts), full)


def test_selfalign_gradient_zero_and_identity_solve():
    d = F.load("pinhole_small")
    pyr = F.pyramids(d)[0]
    gt = P.Pose(np.eye(3), [-0.4, 0.2, -0.5])
    nodes = [P.FrameNode(0, gt, pyr, 0.0), P.FrameNode(1, gt, pyr, 0.1)]
    prob = P.BAProblem(P.MatchGraph(nodes, [P.Edge(0, 1, P.COVISIBILITY)]))
    lv = _level([prob], 0)
    rows, _ = P.se3.pose_rows([gt, gt])
    rec = lv.linearize(_rows(rows)).cpu().numpy()
    assert np.max(np.abs(rec[0, 78:90])) < 1e-10
    res = P.solve_hierarchical(prob)
    assert np.allclose(res.poses[1].matrix(), gt.matrix(), atol=1e-9)


def test_under_constrained_raises():
    prob, gt, guess = _room_problem(n=4)
    prob.graph.edges = [e for e in prob.graph.edges if 3 not in (e.i, e.j)]
    with pytest.raises(P.UnderConstrainedError):
        P.solve_hierarchical(prob)


# ---------------------------------------------------------------------------
# K3 / K4 kernels in isolation
# ---------------------------------------------------------------------------
def _dense_solve(H, b, lam, env=None):
    from paper_2303_16878_b200 import native as N

    lib = N.load()
    dim = H.shape[0]
    Ht, bt = _rows(H), _rows(b)
    work = torch.empty(int(lib.pba_solve_work_bytes(dim)), dtype=torch.uint8, device="cuda")
    delta = torch.zeros(dim, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    env_p = None if env is None else env.ctypes.data
    N.check(lib.pba_solve_dense(Ht.data_ptr(), bt.data_ptr(), dim, lam, env_p, work.data_ptr(),
                                delta.data_ptr(), status.data_ptr(),
                                torch.cuda.current_stream().cuda_stream), "solve")
    return delta.cpu().numpy(), int(status.item())


@pytest.mark.parametrize("dim,band", [(1, None), (6, None), (54, None), (63, None), (64, None),
                                      (65, None), (130, None), (594, None), (600, 40),
                                      (1998, 126)])
def test_dense_cholesky_matches_numpy_solve(dim, band):
    """dim <= 64 runs the one-CTA small solve (c1), larger ones the tiled
    factorisation."""
    rng = np.random.default_rng(dim)
    A = rng.normal(size=(dim, dim))
    if band is not None:
        A = np.triu(np.tril(A, band), -band)
    H = A @ A.T + 1e-3 * np.eye(dim)
    b = rng.normal(size=dim)
    lam = 1e-3
    ref = np.linalg.solve(H + lam * np.diag(np.diag(H)), -b)
    x, st = _dense_solve(H, b, lam)
    assert st == 0
    assert np.max(np.abs(x - ref)) <= 1e-8 * np.max(np.abs(ref))
    if band is not None:  # envelope-restricted factorisation gives the same answer
        T = (dim + 63) // 64
        first = np.array([np.nonzero(H[r, : r + 1])[0][0] for r in range(dim)])
        env = np.array([first[t * 64: (t + 1) * 64].min() // 64 for t in range(T)], np.int32)
        x2, st = _dense_solve(H, b, lam, env)
        assert st == 0
        assert np.max(np.abs(x2 - ref)) <= 1e-8 * np.max(np.abs(ref))


def _band_env(H):
    dim = H.shape[0]
    T = (dim + 63) // 64
    first = np.array([(np.nonzero(H[r, : r + 1])[0][:1].tolist() or [r])[0] for r in range(dim)])
    return np.array([first[t * 64: (t + 1) * 64].min() // 64 for t in range(T)], np.int32)


@pytest.mark.parametrize("dim,band", [(3000, 40), (2049, 20), (6016, 60), (4000, 90)])
def test_dissected_cholesky_matches_numpy_solve(dim, band):
    """Narrow tile bands over many tiles take the nested-dissection path
    (segments batched, separators last, padded to whole tiles)."""
    rng = np.random.default_rng(dim + band)
    A = np.triu(np.tril(rng.normal(size=(dim, dim)), band), -band)
    H = A @ A.T + 1e-3 * np.eye(dim)
    b = rng.normal(size=dim)
    lam = 1e-3
    ref = np.linalg.solve(H + lam * np.diag(np.diag(H)), -b)
    env = _band_env(H)
    T = len(env)
    assert max(k - e for k, e in enumerate(env)) <= 3 and T >= 24  # qualifies
    x, st = _dense_solve(H, b, lam, env)
    assert st == 0
    assert np.max(np.abs(x - ref)) <= 1e-8 * np.max(np.abs(ref))


def test_dissected_cholesky_reports_singular():
    dim = 3000
    H = np.eye(dim) + np.diag(np.full(dim - 1, 0.1), -1) + np.diag(np.full(dim - 1, 0.1), 1)
    H[1700, :] = 0.0
    H[:, 1700] = 0.0
    _, st = _dense_solve(H, np.ones(dim), 1e-3, _band_env(H))
    assert st == 1


@pytest.mark.parametrize("dim", [12, 200])
def test_dense_cholesky_reports_singular(dim):
    H = np.eye(dim)
    H[5, 5] = 0.0
    _, st = _dense_solve(H, np.ones(dim), 1e-3)
    assert st == 1
    # the status word is rewritten by the next (good) solve
    x, st = _dense_solve(np.eye(dim) * 2.0, np.ones(dim), 0.0)
    assert st == 0 and np.allclose(x, -0.5)


def test_apply_step_matches_host_boxplus():
    from paper_2303_16878_b200 import native as N

    lib = N.load()
    rng = np.random.default_rng(5)
    n, gauge = 7, 2
    poses = [P.exp(P.PerturbationVector(rng.uniform(-1, 1, 3), rng.uniform(-0.3, 0.3, 3)))
             for _ in range(n)]
    rows, gens = P.se3.pose_rows(poses)
    gens[4] = 999
    delta = rng.uniform(-0.1, 0.1, 6 * (n - 1))
    out = torch.zeros((n, 12), dtype=torch.float64, device="cuda")
    gout = torch.zeros(n, dtype=torch.int32, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    gin = torch.from_numpy(gens).cuda()
    rows_t, delta_t = _rows(rows), _rows(delta)  # keep alive across the async launch
    N.check(lib.pba_apply_step(rows_t.data_ptr(), gin.data_ptr(), delta_t.data_ptr(), n,
                               gauge, out.data_ptr(), gout.data_ptr(), st.data_ptr(),
                               torch.cuda.current_stream().cuda_stream), "apply")
    got, g = out.cpu().numpy(), gout.cpu().numpy()
    assert st.item() == 0
    s = 0
    for k in range(n):
        if k == gauge:
            assert np.array_equal(got[k], rows[k]) and g[k] == gens[k]
            continue
        ref = P.boxplus(P.Pose(poses[k].rotation, poses[k].translation, int(gens[k])),
                        P.PerturbationVector.from_vector(delta[6 * s:6 * s + 6]))
        assert np.allclose(got[k], ref.as_row(), atol=1e-14, rtol=0)
        assert g[k] == ref.generation
        s += 1
    bad = delta.copy()
    bad[3:6] = [0.8, 0.6, 0.1]
    bad_t = _rows(bad)
    N.check(lib.pba_apply_step(rows_t.data_ptr(), gin.data_ptr(), bad_t.data_ptr(), n,
                               gauge, out.data_ptr(), gout.data_ptr(), st.data_ptr(),
                               torch.cuda.current_stream().cuda_stream), "apply")
    assert st.item() == 1


def test_smoke_entry():
    import __graft_entry__

    __graft_entry__.smoke()


def test_table_atan2_matches_numpy():
    """The division-free table atan2 of the spherical projection: absolute error
    within ~1 ulp of pi against a long-double reference (what u = fx*az + cx
    needs), correctly rounded for angles away from 0, exact special values."""
    from paper_2303_16878_b200 import native as N

    lib = N.load()
    rng = np.random.default_rng(9)
    n = 1 << 20
    mag = 10.0 ** rng.uniform(-6, 3, n)
    ang = rng.uniform(-math.pi, math.pi, n)
    x = mag * np.cos(ang)
    y = mag * np.sin(ang) * 10.0 ** rng.uniform(-3, 3, n)
    special = np.array([[0.0, 1.0], [0.0, -1.0], [1.0, 0.0], [-1.0, 0.0], [-0.0, -1.0],
                        [1e-300, -1.0], [-1e-300, -1.0], [0.0, 0.0], [-0.0, 0.0], [3.0, 1e-320]])
    y = np.concatenate([y, special[:, 0]])
    x = np.concatenate([x, special[:, 1]])
    yt, xt = _rows(y), _rows(x)
    out = torch.empty_like(yt)
    N.check(lib.pba_atan2_batch(yt.data_ptr(), xt.data_ptr(), y.size, out.data_ptr(),
                                torch.cuda.current_stream().cuda_stream), "atan2")
    got = out.cpu().numpy()
    ref_ld = np.arctan2(y.astype(np.longdouble), x.astype(np.longdouble))
    cr = ref_ld.astype(np.float64)
    err = np.abs(got.astype(np.longdouble) - ref_ld).astype(np.float64)
    assert float(err.max()) <= np.spacing(math.pi), float(err.max())
    big = np.abs(cr) > 0.1
    assert np.mean(got[big] == cr[big]) > 0.998
    ref = np.arctan2(y, x)
    assert np.array_equal(np.signbit(got[-10:]), np.signbit(ref[-10:]))
    assert np.array_equal(got[-10:], ref[-10:])

# ---------------------------------------------------------------------------
# reference test cases (pkg/tests/test_solver.py) restated on the device path
# ---------------------------------------------------------------------------
def _affine_image(cam, rng):
    """test_solver.py:59-77: channels affine in pixel coordinates."""
    h, w = cam.height, cam.width
    cols, rows = np.meshgrid(np.arange(w, dtype=float), np.arange(h, dtype=float))
    a = rng.uniform(-0.01, 0.01, 2)
    b = rng.uniform(-0.02, 0.02, 2)
    normals = np.zeros((h, w, 3))
    base = np.array([0.1, -0.15, -0.97])
    for k in range(3):
        c = rng.uniform(-0.003, 0.003, 2)
        normals[..., k] = base[k] + c[0] * cols + c[1] * rows
    return P.CueImage(0.5 + a[0] * cols + a[1] * rows, 3.0 + b[0] * cols + b[1] * rows, normals, cam)


def _pair_problem(src, dst, x_i, x_j):
    nodes = [P.FrameNode(0, x_i, P.CuePyramid((src,), (1.0,)), 0.0),
             P.FrameNode(1, x_j, P.CuePyramid((dst,), (1.0,)), 0.1)]
    return P.BAProblem(P.MatchGraph(nodes, [P.Edge(0, 1, P.COVISIBILITY)]))


def test_all_invalid_destination_kills_all_blocks():
    """test_solver.py:330-339."""
    cam = P.Intrinsics(100.0, 95.0, 32.0, 24.0, 64, 48, P.PINHOLE, 0.1, 50.0)
    src = _affine_image(cam, np.random.default_rng(46))
    dead = P.CueImage(src.intensity.copy(), np.zeros_like(src.depth), np.zeros_like(src.normals), cam)
    prob = _pair_problem(src, dead, P.Pose.identity(), P.Pose.identity())
    rec = _level([prob], 0).linearize(_rows(P.se3.pose_rows([P.Pose.identity()] * 2)[0])).cpu().numpy()
    assert rec[0, 91] == 0 and np.all(rec[0] == 0.0)
    assert P.total_error(prob, level=0) == (0.0, 0)


def test_intensity_offset_shows_in_cost():
    """test_solver.py:154-165: a +0.1 intensity offset gives residual -0.1 on every
    valid block; with Huber delta 0.1 each block costs 0.1^2 (the <= branch)."""
    cam = P.Intrinsics(100.0, 95.0, 32.0, 24.0, 64, 48, P.PINHOLE, 0.1, 50.0)
    src = _affine_image(cam, np.random.default_rng(44))
    dst = P.CueImage(src.intensity + 0.1, src.depth.copy(), src.normals.copy(), cam)
    prob = _pair_problem(src, dst, P.Pose.identity(), P.Pose.identity())
    cost, count = P.total_error(prob, level=0)
    assert count > 0
    assert abs(cost - count * 0.1 ** 2) <= 1e-9 * cost
    o_cost, o_count = O.total_error(prob, [P.Pose.identity()] * 2, 0, P.SolverConfig())
    assert count == o_count and abs(cost - o_cost) <= 1e-12 * o_cost


def test_gauge_invariance_of_device_objective():
    """test_solver.py:423-440 / test_acceptance.py:138-155 on the device cost path."""
    prob, gt, guess = _room_problem(n=5)
    rng = np.random.default_rng(49)
    f_ref, n_ref = P.total_error(prob, level=0)
    for _ in range(5):
        g = P.exp(P.PerturbationVector(rng.uniform(-2, 2, 3), rng.uniform(-0.4, 0.4, 3)))
        moved = [g.compose(n.pose_guess) for n in prob.graph.nodes]
        f_g, n_g = P.total_error(prob, moved, level=0)
        assert n_g == n_ref
        assert abs(f_g - f_ref) / f_ref < 1e-9


def test_solve_level_matches_oracle_level_solve():
    prob, gt, guess = _room_problem(n=6, scales=(0.5, 1.0))
    poses, records = P.solve_level(prob, guess, 1, max_iterations=4)
    rows, gens = P.se3.pose_rows(guess)
    lp = O.OracleLevel([prob], 1, P.SolverConfig())
    o_rows, _, o_recs = O.solve_level_multi(lp, rows, gens.astype(np.int64), 1, P.SolverConfig(), 4)
    assert [(r.iteration, r.accepted, r.valid_blocks) for r in records] == [
        (r.iteration, r.accepted, r.valid_blocks) for r in o_recs]
    er, et = _pose_err(np.stack([p.as_row() for p in poses]), o_rows)
    assert er <= 1e-5 and et <= 1e-5


def test_reference_objects_accepted_duck_typed():
    """Drop-in: objects that merely look like the reference types work."""
    from types import SimpleNamespace as NS

    d = F.load("pinhole_small")
    prob, _ = F.single_problem(d)
    nodes = [NS(id=n.id, pose_guess=NS(rotation=n.pose_guess.rotation,
                                       translation=n.pose_guess.translation, generation=0),
                pyramid=NS(levels=n.pyramid.levels, scales=n.pyramid.scales,
                           __len__=lambda: 1), timestamp=n.timestamp, sensor_id=n.sensor_id)
             for n in prob.graph.nodes]

    class Pyr:
        def __init__(self, p):
            self.levels, self.scales = p.levels, p.scales

        def __len__(self):
            return len(self.levels)

    for n, orig in zip(nodes, prob.graph.nodes):
        n.pyramid = Pyr(orig.pyramid)
    duck = NS(graph=NS(nodes=nodes, edges=prob.graph.edges), gauge_index=0,
              extrinsics_of=prob.extrinsics_of)
    res = P.solve_hierarchical(duck)
    _check_trace(res.records, d["trace"])


def test_invalid_level_schedule_and_fusion_errors():
    d = F.load("pinhole_small")
    prob, _ = F.single_problem(d)
    with pytest.raises(ValueError):
        P.solve_hierarchical(prob, levels=[3])
    probs = F.fusion_problems(F.load("fusion_small"))
    probs[1].graph.nodes.append(probs[1].graph.nodes[1])
    with pytest.raises(P.FusionConfigError):
        P.solve_fusion(probs[0], probs[1], "coupled")
    with pytest.raises(ValueError):
        P.solve_fusion(probs[0], probs[0], "sideways")


@pytest.mark.parametrize("model", ["pinhole", "spherical"])
def test_self_projection_counts_match_oracle(model):
    """Identity poses put every sample on an integer pixel, where floor() is
    decided by the last bit of the projected coordinate.  Pinhole u, v are a
    multiply, an IEEE division and an add, so they reproduce the reference bit
    for bit.  Spherical u, v go through atan2, whose last bit is
    implementation-defined: numpy's SIMD arctan2 and libm's atan2 (the oracle)
    already disagree on this input (reference 2732 vs oracle 2731 blocks in
    the first trial), so the device is held to the same +-1 block per pair."""
    rng = np.random.default_rng(7)
    if model == "pinhole":
        cam = P.Intrinsics(100.0, 95.0, 32.0, 24.0, 64, 48, P.PINHOLE, 0.1, 50.0)
    else:
        cam = P.Intrinsics(64 / (2 * math.pi), 48 / (math.pi / 2), 32.0, 24.0, 64, 48,
                           P.SPHERICAL, 0.1, 50.0)
    for trial in range(3):
        src = _affine_image(cam, rng)
        prob = _pair_problem(src, src, P.Pose.identity(), P.Pose.identity())
        for tol in (None, float("inf")):
            rows = P.se3.pose_rows([P.Pose.identity()] * 2)[0]
            got = _level([prob], 0, tolerance_override=tol).linearize(_rows(rows)).cpu().numpy()
            lp = O.OracleLevel([prob], 0, P.SolverConfig())
            if tol is not None:
                lp.with_tolerance(tol)
            ref = lp.records(rows)
            if model == "pinhole":
                F.compare_records(got, ref)
            else:
                assert abs(got[0, 91] - ref[0, 91]) <= 1
                assert abs(got[0, 90] - ref[0, 90]) <= 1e-18 * ref[0, 91] + 1e-6 * ref[0, 90]
                assert F.rel(got[0, :78], ref[0, :78]) <= 2.0 / ref[0, 91]  # one block's share


# ---------------------------------------------------------------------------
# K5: GPU overlap counting in build_graph
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", CASES)
def test_build_graph_gpu_equals_reference_edges(name):
    d = F.load(name)
    pyrs = F.pyramids(d)
    guess = F.poses(d["guess"])
    nodes = [P.FrameNode(k, guess[k], pyrs[k], 0.1 * k) for k in range(len(pyrs))]
    ext = P.SensorExtrinsics(P.Pose.from_row(d["ext"]))
    g = P.build_graph(nodes, extrinsics=ext, device="cuda:0")
    assert [(e.i, e.j) for e in g.edges] == [tuple(map(int, e)) for e in d["edges"]]
    assert [e.kind == P.COVISIBILITY for e in g.edges] == list(d["edge_kinds"])


def test_build_graph_gpu_equals_host_on_corridor():
    import bench

    problems, guess, gt, meta = bench.build_problem("c4", torch.device("cuda", 0), 60)
    prob = problems[0]
    nodes = prob.graph.nodes
    ext = prob.extrinsics_of("sensor0")
    crit = P.MatchCriteria(max_translation=40.0)
    g_host = P.build_graph(nodes, crit, extrinsics=ext, threads=8)
    assert prob.graph.edges == g_host.edges  # bench built it on the device
    assert len(g_host.edges) == 968  # SURVEY.md App. C validated prototype


_NCCL_SCRIPT = r"""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.distributed as dist
import paper_2303_16878_b200 as P
from tests import fixtures as F
d = F.load("pinhole_small")
prob, _ = F.single_problem(d)
out = {}
pcg = P.SolverConfig(linear_solver="pcg")
res = P.solve_hierarchical(prob, P.SolverConfig())
out["plain"] = [list(p.as_row()) for p in res.poses]
out["plain_pcg"] = [list(p.as_row()) for p in P.solve_hierarchical(prob, pcg).poses]
os.environ["PBA_FORCE_SHARDED"] = "1"
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
res = P.solve_hierarchical(prob, P.SolverConfig())
out["nccl"] = [list(p.as_row()) for p in res.poses]
out["trace"] = [(r.level, r.iteration, r.accepted, r.valid_blocks) for r in res.records]
out["nccl_pcg"] = [list(p.as_row()) for p in P.solve_hierarchical(prob, pcg).poses]
dist.destroy_process_group()
print(json.dumps(out))
"""


def test_sharded_path_over_nccl_matches_single_gpu():
    """The multi-GPU code path (ShardedLevel: record all_gather, pose and
    scalar broadcasts over NCCL) on one rank gives bit-identical poses."""
    import json
    import os
    import subprocess
    import sys

    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29517")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _NCCL_SCRIPT], cwd=root, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert np.array_equal(np.array(out["plain"]), np.array(out["nccl"]))
    assert np.array_equal(np.array(out["plain_pcg"]), np.array(out["nccl_pcg"]))  # rank-0 PCG
    assert len(out["trace"]) > 0


def test_os0_128_full_resolution_records_and_trace_match_oracle():
    """The bench's sensor shape (OS0-128, 128x1024, K6-estimated normals,
    8192-pixel chunks): per-pair records at full resolution and a short LM
    trace against the oracle."""
    import bench

    problems, guess, gt, meta = bench.build_problem("c4", torch.device("cuda", 0), 5)
    prob = problems[0]
    level = meta["level"]
    rows, _ = P.se3.pose_rows(guess)
    got = _level([prob], level).linearize(_rows(rows)).cpu().numpy()
    ref = O.OracleLevel([prob], level, P.SolverConfig()).records(rows)
    F.compare_records(got, ref)
    assert ref[:, 91].sum() > 1e5
    poses, records = P.solve_level(prob, guess, level, max_iterations=3)
    lp = O.OracleLevel([prob], level, P.SolverConfig())
    gens = np.zeros(len(guess), np.int64)
    o_rows, _, o_recs = O.solve_level_multi(lp, rows, gens, level, P.SolverConfig(), 3)
    assert [(r.iteration, r.accepted, r.valid_blocks) for r in records] == [
        (r.iteration, r.accepted, r.valid_blocks) for r in o_recs]
    for a, b in zip(records, o_recs):
        assert a.lam == b.lam
        assert abs(a.error - b.error) <= 1e-6 * b.error
    er, et = _pose_err(np.stack([p.as_row() for p in poses]), o_rows)
    assert er <= 1e-5 and et <= 1e-5


def test_c4_full_size_properties():
    """BASELINE's c4 at full size (1000 OS0-128 scans, ~19k pairs), where the
    oracle is too slow: records bit-identical across launches and across a
    3-way pair sharding (so 1/2/4/8 GPUs give identical results), assembled
    totals equal to the record sums, and a sampled pair equal to the oracle."""
    import bench

    dev = torch.device("cuda", 0)
    problems, guess, gt, meta = bench.build_problem("c4", dev)
    prob = problems[0]
    level = meta["level"]
    n = len(prob.graph.edges)
    assert n > 18000
    rows, gens = P.se3.pose_rows(guess)
    lv = _level([prob], level)
    full = lv.linearize(_rows(rows)).cpu().numpy()
    assert np.array_equal(full, lv.linearize(_rows(rows)).cpu().numpy())
    cuts = [0, n // 3, (2 * n) // 3, n]
    parts = [_level([prob], level, pair_range=(a, b), assemble=False).linearize(_rows(rows))
             .cpu().numpy() for a, b in zip(cuts, cuts[1:])]
    assert np.array_equal(np.concatenate(parts), full)
    lv.set_poses(rows, gens)
    cost, count = lv.evaluate_current()
    assert count == int(full[:, 91].sum())
    assert abs(cost - full[:, 90].sum()) <= 1e-12 * cost
    k = n // 2
    sub = P.BAProblem(P.MatchGraph(prob.graph.nodes, prob.graph.edges[k:k + 1]), prob.extrinsics)
    ref = O.OracleLevel([sub], level, P.SolverConfig()).records(rows)
    F.compare_records(full[k:k + 1], ref)


@pytest.mark.parametrize("name", CASES)
def test_records_agree_far_below_the_bar(name):
    """The SURVEY bar is 1e-5; the device records actually agree with the
    oracle and with the reference's own records to ~1e-13 relative (fp64
    rounding of a different but exact algebra), counts exactly."""
    d = F.load(name)
    prob, _ = F.single_problem(d)
    rows = d["guess"]
    for l in range(len(d["scales"])):
        got = _level([prob], l).linearize(_rows(rows)).cpu().numpy()
        ref = O.OracleLevel([prob], l, P.SolverConfig()).records(rows)
        gold = d[f"rec_guess_{l}"]
        for other in (ref, gold):
            for sl in (slice(0, 78), slice(78, 90), slice(90, 91)):
                scale = max(np.abs(other[:, sl]).max(), 1e-300)
                assert np.abs(got[:, sl] - other[:, sl]).max() <= 1e-11 * scale
            assert np.array_equal(got[:, 91], other[:, 91])


def test_chunk_launch_order_does_not_change_records(monkeypatch):
    """Partials are slot-addressed, so every CTA launch order (edge order,
    destination- or source-interleaved) gives bit-identical records."""
    prob, gt, guess = _room_problem()
    rows, _ = P.se3.pose_rows(guess)
    out = {}
    for order in ("pair", "dst", "src", "blk"):
        monkeypatch.setenv("PBA_CHUNK_ORDER", order)
        monkeypatch.setenv("PBA_CHUNK_BLOCK", "3")
        out[order] = _level([prob], 0).linearize(_rows(rows)).cpu().numpy()
    for order in ("dst", "src", "blk"):
        assert np.array_equal(out["pair"], out[order]), order


@pytest.mark.parametrize("model", ["pinhole", "spherical"])
def test_tiled_walk_and_partial_bands_match_oracle(monkeypatch, model):
    """Chunks of whole 8-row bands walked in 16 x 8 tiles (linearize.cu
    pair_chunk_pixels), here 16-row bands of a 100-row image so each pair
    also ends in a partial 4-row band walked row-major: records within the
    §8(c) bar of the oracle, and equal to the all-row-major chunking up to
    summation order (counts exactly)."""
    from paper_2303_16878_b200 import scenes as S

    if model == "pinhole":
        cam = P.Intrinsics(120.0, 120.0, 79.5, 49.5, 160, 100, P.PINHOLE, 0.1, 50.0)
        prob, gt, guess = _room_problem(n=4, cam=cam)
    else:
        cam = S.hdl64(256, 100)
        gt = S.corridor_trajectory(4, 0.5)
        pyrs = S.host_pyramids(S.corridor_scene(20.0), cam, gt, P.Pose.identity(), (1.0,))
        guess = S.perturb(gt, 0.05, math.radians(2.0), 11)
        nodes = [P.FrameNode(k, guess[k], pyrs[k], 0.1 * k) for k in range(len(gt))]
        prob = P.BAProblem(P.build_graph(nodes))
    rows, _ = P.se3.pose_rows(guess)
    width = cam.width
    monkeypatch.setenv("PBA_CHUNK_UNITS", str(16 * width // 256))  # 16-row bands
    lv = _level([prob], 0)
    assert lv.chunk_pixels == 16 * width
    tiled = lv.linearize(_rows(rows)).cpu().numpy()
    ref = O.OracleLevel([prob], 0, P.SolverConfig()).records(rows)
    F.compare_records(tiled, ref)
    monkeypatch.setenv("PBA_CHUNK_UNITS", "1")  # 256-pixel chunks: row-major everywhere
    flat = _level([prob], 0).linearize(_rows(rows)).cpu().numpy()
    assert np.array_equal(tiled[:, 91], flat[:, 91])
    np.testing.assert_allclose(tiled[:, :91], flat[:, :91], rtol=1e-11,
                               atol=1e-11 * np.abs(flat[:, :91]).max())


@pytest.mark.parametrize("config,frames", [("c3", 4), ("c5", 3)])
def test_bench_shapes_records_and_trace_match_oracle(config, frames):
    """The other bench sensor shapes at full resolution against the oracle:
    c3 (640x480 pinhole on a forward-looking mount) and c5 (coupled OS0-128
    spherical + 640x480 pinhole in one level problem) — per-pair records of
    the finest level at the perturbed guess and a short LM trace."""
    import bench

    problems, guess, gt, meta = bench.build_problem(config, torch.device("cuda", 0), frames)
    level = meta["level"]
    rows, gens = P.se3.pose_rows(guess)
    assert sum(len(p.graph.edges) for p in problems) > 0
    got = _level(problems, level).linearize(_rows(rows)).cpu().numpy()
    ref = O.OracleLevel(problems, level, P.SolverConfig()).records(rows)
    F.compare_records(got, ref)
    assert ref[:, 91].sum() > 1e4
    from paper_2303_16878_b200.bundle import _lm_level, _Runtime

    backend = _Runtime().level(problems, level, P.SolverConfig())
    backend.set_poses(rows, gens)
    records = _lm_level(backend, level, P.SolverConfig(), 3)
    lp = O.OracleLevel(problems, level, P.SolverConfig())
    _, _, o_recs = O.solve_level_multi(lp, rows, gens.astype(np.int64), level, P.SolverConfig(), 3)
    assert [(r.iteration, r.accepted, r.valid_blocks, r.lam) for r in records] == [
        (r.iteration, r.accepted, r.valid_blocks, r.lam) for r in o_recs]
    for a, b in zip(records, o_recs):
        assert abs(a.error - b.error) <= 1e-6 * b.error
