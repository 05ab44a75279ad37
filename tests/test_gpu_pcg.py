"""K3b block-Jacobi PCG (App. C c3, `SolverConfig(linear_solver="pcg")`):
the kernel against numpy's exact solve on block-sparse SPD systems, the
singular report, and the LM trace through the public API against the
reference's goldens and the oracle (PCG run to 1e-12 gives the exact step
to far inside the 1e-6 trace bar)."""
import math

import numpy as np
import pytest

import paper_2303_16878_b200 as P
from oracle import oracle as O
from paper_2303_16878_b200.device import block_rows
from tests import fixtures as F
from tests.test_gpu_parity import CASES, _check_trace, _pose_err, _room_problem

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _pcg(H, b, lam, row_ptr, cols, max_iter=5000, tol=1e-14):
    from paper_2303_16878_b200 import native as N

    lib = N.load()
    n_free = H.shape[0] // 6
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    Ht, bt, rp, cc = dev(H.astype(np.float64)), dev(b.astype(np.float64)), dev(row_ptr), dev(cols)
    work = torch.empty(int(lib.pba_pcg_work_bytes(n_free)), dtype=torch.uint8, device="cuda")
    delta = torch.full((6 * n_free,), np.nan, dtype=torch.float64, device="cuda")
    status = torch.full((1,), 7, dtype=torch.int32, device="cuda")
    info = torch.zeros(3, dtype=torch.float64, device="cuda")
    N.check(lib.pba_solve_pcg(Ht.data_ptr(), bt.data_ptr(), n_free, lam, rp.data_ptr(),
                              cc.data_ptr(), max_iter, tol, work.data_ptr(), delta.data_ptr(),
                              status.data_ptr(), info.data_ptr(),
                              torch.cuda.current_stream().cuda_stream), "pba_solve_pcg")
    return delta.cpu().numpy(), int(status.item()), info.cpu().numpy()


def _graph_system(n_poses, edges, seed, gauge=0):
    """A normal matrix with the block pattern of a pose graph: every edge
    adds J^T J of a random 6x12 Jacobian (like a pair record), gauge removed."""
    rng = np.random.default_rng(seed)
    H = np.zeros((6 * n_poses, 6 * n_poses))
    for i, j in edges:
        J = rng.normal(size=(24, 12))
        blk = J.T @ J
        idx = np.r_[6 * i: 6 * i + 6, 6 * j: 6 * j + 6]
        H[np.ix_(idx, idx)] += blk
    keep = np.array([k for k in range(6 * n_poses) if k // 6 != gauge])
    slot = np.array([-1 if k == gauge else k - (k > gauge) for k in range(n_poses)], np.int32)
    pi = np.array([e[0] for e in edges], np.int32)
    pj = np.array([e[1] for e in edges], np.int32)
    row_ptr, cols = block_rows(slot, pi, pj)
    return H[np.ix_(keep, keep)], row_ptr, cols, rng.normal(size=keep.size)


def _corridor_edges(n, reach):
    return [(i, j) for i in range(n) for j in range(i + 1, min(n, i + reach + 1))]


@pytest.mark.parametrize("n,reach,lam", [(10, 3, 1e-3), (200, 20, 1e-3), (1000, 20, 1e-3),
                                         (300, 5, 1e-6)])
def test_pcg_matches_numpy_solve(n, reach, lam):
    H, rp, cols, b = _graph_system(n, _corridor_edges(n, reach), seed=n + reach)
    ref = np.linalg.solve(H + lam * np.diag(np.diag(H)), -b)
    x, st, info = _pcg(H, b, lam, rp, cols)
    assert st == 0 and info[2] == 1.0, info
    assert np.max(np.abs(x - ref)) <= 1e-9 * np.max(np.abs(ref)), info


def test_pcg_general_graph_and_determinism():
    rng = np.random.default_rng(3)
    n = 400
    edges = sorted({tuple(sorted(rng.choice(n, 2, replace=False))) for _ in range(3000)}
                   | {(k, k + 1) for k in range(n - 1)})
    H, rp, cols, b = _graph_system(n, edges, seed=4)
    ref = np.linalg.solve(H + 1e-3 * np.diag(np.diag(H)), -b)
    x1, st, info = _pcg(H, b, 1e-3, rp, cols)
    x2, _, _ = _pcg(H, b, 1e-3, rp, cols)
    assert st == 0 and info[2] == 1.0
    assert np.array_equal(x1, x2)  # fixed reduction order: bit-identical reruns
    assert np.max(np.abs(x1 - ref)) <= 1e-9 * np.max(np.abs(ref))


def test_pcg_iteration_cap_returns_the_iterate():
    H, rp, cols, b = _graph_system(200, _corridor_edges(200, 20), seed=9)
    x, st, info = _pcg(H, b, 1e-3, rp, cols, max_iter=3, tol=1e-14)
    assert st == 0 and info[0] == 3 and info[2] == 0.0 and np.isfinite(x).all()
    assert 0.0 < info[1] < 1.0  # residual reduced but not converged


def test_pcg_reports_singular_and_zero_rhs():
    H, rp, cols, b = _graph_system(20, _corridor_edges(20, 2), seed=1)
    Hs = H.copy()
    Hs[30:36, :] = 0.0
    Hs[:, 30:36] = 0.0
    _, st, _ = _pcg(Hs, b, 1e-3, rp, cols)
    assert st == 1
    x, st, info = _pcg(H, np.zeros_like(b), 1e-3, rp, cols)
    assert st == 0 and info[0] == 0 and not x.any()


@pytest.mark.parametrize("name", CASES)
def test_pcg_lm_trace_matches_reference(name):
    d = F.load(name)
    prob, _ = F.single_problem(d)
    res = P.solve_hierarchical(prob, P.SolverConfig(linear_solver="pcg"))
    _check_trace(res.records, d["trace"])
    er, et = _pose_err(np.stack([p.as_row() for p in res.poses]), d["final"])
    assert er <= 1e-5 and et <= 1e-5


def test_pcg_config1_trace_matches_oracle():
    prob, gt, guess = _room_problem()
    res = P.solve_hierarchical(prob, P.SolverConfig(linear_solver="pcg"))
    final_o, recs_o = O.hierarchical([prob], P.SolverConfig())
    assert [(r.level, r.iteration, r.accepted, r.valid_blocks, r.lam) for r in res.records] == [
        (r.level, r.iteration, r.accepted, r.valid_blocks, r.lam) for r in recs_o]
    for a, b in zip(res.records, recs_o):
        assert abs(a.error - b.error) <= 1e-6 * b.error
    er, et = _pose_err(np.stack([p.as_row() for p in res.poses]), final_o)
    assert er <= 1e-5 and et <= 1e-5
    assert math.isfinite(res.records[-1].error)


def test_reference_style_config_without_b200_fields():
    """A config object with only the reference SolverConfig fields (as
    photoba.solver.SolverConfig has) still solves, with the exact solver."""
    import dataclasses
    import types

    extra = {"linear_solver", "pcg_max_iterations", "pcg_tolerance"}
    ref_cfg = types.SimpleNamespace(**{f.name: getattr(P.SolverConfig(), f.name)
                                       for f in dataclasses.fields(P.SolverConfig)
                                       if f.name not in extra})
    d = F.load(CASES[0])
    prob, _ = F.single_problem(d)
    res = P.solve_hierarchical(prob, ref_cfg)
    _check_trace(res.records, d["trace"])
