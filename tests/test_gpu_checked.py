"""Stand-ins for compute-sanitizer, which is closed on this
GPU pool (`gpurun` refuses it: runs under it left GPUs needing a reset).

* memcheck -> the bounds-checked library (libpba_b200_checked.so, built
  with -DPBA_CHECKED): device index assertions on the source texel, ray
  table and destination-corner gathers and the partial slot of K1, the H
  writes of the assembly and the block columns of the PCG mat-vec.  The
  sanitizer workload (tools/sanitize_case.py: c1 with Cholesky and PCG, a
  5-scan OS0-128 problem through K5/K6/K1-K4, the dissected Cholesky, atan2
  and raster decode) runs on it and must print no PBA_CHECK line.
* racecheck / synccheck -> determinism under repetition: a shared-memory
  race or a missing barrier in the reductions (K1's warp reduce-scatter and
  cross-warp sum, the totals tree, the cooperative PCG's grid-wide dot
  products) shows up as run-to-run differences, so every such kernel is
  rerun and compared bit for bit.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2303_16878_b200 as P

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_sanitizer_workload_on_bounds_checked_library():
    env = dict(os.environ, PBA_CHECKED="1")
    r = subprocess.run([sys.executable, "tools/sanitize_case.py"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "sanitize case ok" in r.stdout
    assert "checked library: 1" in r.stdout  # the -DPBA_CHECKED build really ran
    bad = [ln for ln in r.stdout.splitlines() if ln.startswith("PBA_CHECK")]
    assert not bad, bad[:10]


def test_reductions_bit_identical_under_repetition():
    import bench
    from paper_2303_16878_b200.device import DeviceLevel, FrameStore

    dev = torch.device("cuda", 0)
    problems, guess, _, meta = bench.build_problem("c4", dev, 24)
    level = meta["level"]
    rows, gens = P.se3.pose_rows(guess)
    store = FrameStore(dev)
    for solver in ("cholesky", "pcg"):
        lv = DeviceLevel(problems, level, P.SolverConfig(linear_solver=solver), store)
        first = None
        for _ in range(6):
            lv.set_poses(rows, gens)
            c0, n0 = lv.evaluate_current()
            ok_s, ok_u, c1, n1 = lv.try_step(1e-3)
            out = (lv.records.cpu().numpy().copy(), lv.Hb[0].cpu().numpy().copy(),
                   lv.delta.cpu().numpy().copy(), lv.poses[1].cpu().numpy().copy(), c0, c1)
            assert ok_s and ok_u
            if first is None:
                first = out
                continue
            for a, b in zip(first, out):
                assert np.array_equal(np.asarray(a), np.asarray(b))
