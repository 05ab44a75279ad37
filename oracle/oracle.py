"""ORACLE — test infrastructure only (checker + CPU baseline, never product).

Python driver around the C restatement `pba_oracle.c` of the reference
photometric-BA path.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py` (its CPU-baseline / reference arm) may import this module.

What it restates (reference: /root/reference/pkg/src/photoba):
  derive_image        CueImage.__post_init__                    cues.py:106-147
  OracleLevel         _LevelProblem (contexts, evaluate, apply)  solver.py:393-460
  solve_level_multi   _solve_level_multi (LM loop)              solver.py:495-538
  hierarchical        _hierarchical                             solver.py:585-606
  total_error         total_error                               solver.py:655-670
  boxplus / exp       geometry.py:30-45, 137-143, 202-219
The linear solve is np.linalg.solve, exactly as the reference
(solver.py:510-512).  Parity of the restatement is pinned by
tests/test_oracle_golden.py against vectors produced by the reference.

Poses are plain (R, t) numpy pairs; problems are duck-typed: anything with
`graph.nodes[k].pyramid.levels[l]` exposing intensity/depth/normals/
intrinsics, `graph.edges` with i/j, `extrinsics_of(sensor_id)` and
`gauge_index` (reference objects and the product package's objects both
qualify).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "liboracle.so"
REC = 92

_LAMBDA_CEILING = 1e12          # solver.py:489
_COST_FLOOR_PER_BLOCK = 1e-18   # solver.py:492
_REORTHO_INTERVAL = 1000        # geometry.py:17


def build(force: bool = False) -> Path:
    src = HERE / "pba_oracle.c"
    if not force and LIB_PATH.exists() and LIB_PATH.stat().st_mtime >= src.stat().st_mtime:
        return LIB_PATH
    LIB_PATH.parent.mkdir(exist_ok=True)
    tmp = LIB_PATH.with_suffix(".tmp.so")
    cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
           str(src), "-o", str(tmp), "-lm"]
    subprocess.run(cmd, check=True, capture_output=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


class _Cam(ctypes.Structure):
    _fields_ = [("model", ctypes.c_int32), ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("cx", ctypes.c_double), ("cy", ctypes.c_double), ("dmin", ctypes.c_double),
                ("dmax", ctypes.c_double)]


_DP = ctypes.POINTER(ctypes.c_double)
_BP = ctypes.POINTER(ctypes.c_uint8)


class _Image(ctypes.Structure):
    _fields_ = [("intensity", _DP), ("depth", _DP), ("normals", _DP), ("grad_intensity", _DP),
                ("grad_depth", _DP), ("grad_normals", _DP), ("depth_valid", _BP),
                ("normal_valid", _BP), ("samp_intensity", _BP), ("samp_depth", _BP),
                ("samp_normals", _BP), ("cam", _Cam)]


class _Pair(ctypes.Structure):
    _fields_ = [("i", ctypes.c_int32), ("j", ctypes.c_int32), ("src", ctypes.c_int32),
                ("dst", ctypes.c_int32), ("ext", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("tol", ctypes.c_double)]


class _Cfg(ctypes.Structure):
    _fields_ = [("delta", ctypes.c_double * 3), ("omega", ctypes.c_double * 5),
                ("stride", ctypes.c_int32), ("pad", ctypes.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(str(build()))
        L.oracle_derive.restype = None
        L.oracle_linearize.restype = None
        L.oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(_DP)


def _bp(a):
    return a.ctypes.data_as(_BP)


def cam_struct(intr) -> _Cam:
    model = 0 if intr.model == "pinhole" else 1
    return _Cam(model, int(intr.width), int(intr.height), 0, float(intr.fx), float(intr.fy),
                float(intr.cx), float(intr.cy), float(intr.depth_min), float(intr.depth_max))


@dataclass
class OracleImage:
    """All CueImage fields of one (frame, level), as C-contiguous arrays."""

    intensity: np.ndarray
    depth: np.ndarray
    normals: np.ndarray
    grad_intensity: np.ndarray
    grad_depth: np.ndarray
    grad_normals: np.ndarray
    depth_valid: np.ndarray
    normal_valid: np.ndarray
    sampleable_core: np.ndarray
    sampleable_normals: np.ndarray
    intrinsics: object

    def struct(self) -> _Image:
        return _Image(_dp(self.intensity), _dp(self.depth), _dp(self.normals),
                      _dp(self.grad_intensity), _dp(self.grad_depth), _dp(self.grad_normals),
                      _bp(self.depth_valid), _bp(self.normal_valid), _bp(self.sampleable_core),
                      _bp(self.sampleable_core), _bp(self.sampleable_normals),
                      cam_struct(self.intrinsics))


def derive_image(intensity, depth, normals, intr) -> OracleImage:
    """CueImage.__post_init__ restated in C (cues.py:106-147)."""
    I = np.ascontiguousarray(intensity, dtype=np.float64)
    Din = np.ascontiguousarray(depth, dtype=np.float64)
    Nin = np.ascontiguousarray(normals, dtype=np.float64)
    h, w = I.shape
    if Din.shape != (h, w) or Nin.shape != (h, w, 3):
        raise ValueError("cue channel shapes disagree")
    D = np.empty_like(Din)
    N = np.empty_like(Nin)
    gI = np.empty((h, w, 2))
    gD = np.empty((h, w, 2))
    gN = np.empty((h, w, 3, 2))
    masks = [np.empty((h, w), np.uint8) for _ in range(4)]
    lib().oracle_derive(ctypes.c_int(h), ctypes.c_int(w), ctypes.c_double(intr.depth_min),
                        ctypes.c_double(intr.depth_max), _dp(I), _dp(Din), _dp(Nin), _dp(D),
                        _dp(N), _dp(gI), _dp(gD), _dp(gN), *(_bp(m) for m in masks))
    dv, nv, sc, sn = masks
    return OracleImage(I, D, N, gI, gD, gN, dv, nv, sc, sn, intr)


def image_of(cue) -> OracleImage:
    return derive_image(cue.intensity, cue.depth, cue.normals, cue.intrinsics)


# ---------------------------------------------------------------------------
# SE(3) helpers (geometry.py)
# ---------------------------------------------------------------------------
def quat_to_rotation(qx, qy, qz, qw):
    n = qw * qw + qx * qx + qy * qy + qz * qz
    s = 2.0 / n
    wx, wy, wz = s * qw * qx, s * qw * qy, s * qw * qz
    xx, xy, xz = s * qx * qx, s * qx * qy, s * qx * qz
    yy, yz, zz = s * qy * qy, s * qy * qz, s * qz * qz
    return np.array([[1.0 - (yy + zz), xy - wz, xz + wy],
                     [xy + wz, 1.0 - (xx + zz), yz - wx],
                     [xz - wy, yz + wx, 1.0 - (xx + yy)]])


class OraclePerturbationError(ValueError):
    pass


def boxplus(R, t, gen, v):
    """X * exp(v) with generation bookkeeping (geometry.py:137-143, 202-219)."""
    dq = v[3:]
    nq2 = float(dq @ dq)
    if nq2 >= 1.0:
        raise OraclePerturbationError(f"||dq|| = {math.sqrt(nq2):.6f} >= 1")
    D = quat_to_rotation(dq[0], dq[1], dq[2], math.sqrt(1.0 - nq2))
    R2 = R @ D
    t2 = R @ v[:3] + t
    g2 = gen + 1
    if g2 >= _REORTHO_INTERVAL:
        u, _, vt = np.linalg.svd(R2)
        R2 = u @ vt
        if np.linalg.det(R2) < 0.0:
            u[:, -1] = -u[:, -1]
            R2 = u @ vt
        g2 = 0
    return R2, t2, g2


def pose_arrays(poses):
    """list of pose-like objects -> (N,12) array + generations."""
    arr = np.zeros((len(poses), 12))
    gens = np.zeros(len(poses), np.int64)
    for k, p in enumerate(poses):
        arr[k, :9] = np.asarray(p.rotation, float).reshape(9)
        arr[k, 9:] = np.asarray(p.translation, float).reshape(3)
        gens[k] = getattr(p, "generation", 0)
    return arr, gens


# ---------------------------------------------------------------------------
# _LevelProblem
# ---------------------------------------------------------------------------
class OracleLevel:
    """_LevelProblem restated (solver.py:393-460) on top of the C kernel."""

    def __init__(self, problems, level, cfg, image_cache=None):
        self.cfg = cfg
        self.n_poses = len(problems[0].graph.nodes)
        self.gauge = problems[0].gauge_index
        cache = image_cache if image_cache is not None else {}
        self.images: list[OracleImage] = []
        slot_of = {}
        exts = []
        pairs = []
        for pi_, problem in enumerate(problems):
            nodes = problem.graph.nodes
            index_of = {n.id: k for k, n in enumerate(nodes)}
            for edge in problem.graph.edges:
                ni, nj = nodes[index_of[edge.i]], nodes[index_of[edge.j]]
                if ni.sensor_id != nj.sensor_id:
                    raise ValueError("edges must connect frames of one sensor")
                ext = problem.extrinsics_of(ni.sensor_id)
                scale = ni.pyramid.scales[level]
                tol = cfg.occlusion_depth_tolerance / scale
                slots = []
                for node in (ni, nj):
                    key = (pi_, node.id)
                    if key not in slot_of:
                        cue = node.pyramid.levels[level]
                        ck = (id(cue), level)
                        if ck not in cache:
                            cache[ck] = image_of(cue)
                        slot_of[key] = len(self.images)
                        self.images.append(cache[ck])
                    slots.append(slot_of[key])
                off = ext.offset
                exts.append(np.concatenate([np.asarray(off.rotation, float).reshape(9),
                                            np.asarray(off.translation, float)]))
                pairs.append((index_of[edge.i], index_of[edge.j], slots[0], slots[1],
                              len(exts) - 1, tol))
        self.pairs = pairs
        self.exts = np.ascontiguousarray(np.array(exts).reshape(-1, 12))
        self._img_structs = (_Image * max(len(self.images), 1))(*[im.struct() for im in self.images])
        self._pair_structs = (_Pair * max(len(pairs), 1))(
            *[_Pair(i, j, s, d, e, 0, t) for (i, j, s, d, e, t) in pairs])
        c = _Cfg()
        c.delta[:] = [cfg.huber_delta_intensity, cfg.huber_delta_depth, cfg.huber_delta_normal]
        c.omega[:] = [cfg.omega_intensity, cfg.omega_depth, *cfg.omega_normal]
        c.stride = int(cfg.pixel_stride)
        self._cfg = c

    def with_tolerance(self, tol):
        for k in range(len(self.pairs)):
            self._pair_structs[k].tol = tol
        return self

    def records(self, pose_arr, want_jacobians=True, threads=None, pair_subset=None):
        n = len(self.pairs)
        threads = threads or lib().oracle_max_threads()
        pose_arr = np.ascontiguousarray(pose_arr, dtype=np.float64)
        if pair_subset is not None:
            sub = (_Pair * len(pair_subset))(*[self._pair_structs[k] for k in pair_subset])
            out = np.zeros((len(pair_subset), REC))
            lib().oracle_linearize(self._img_structs, sub, ctypes.c_int(len(pair_subset)),
                                   _dp(pose_arr), _dp(self.exts), ctypes.byref(self._cfg),
                                   ctypes.c_int(int(want_jacobians)), ctypes.c_int(threads),
                                   _dp(out))
            return out
        out = np.zeros((n, REC))
        if n:
            lib().oracle_linearize(self._img_structs, self._pair_structs, ctypes.c_int(n),
                                   _dp(pose_arr), _dp(self.exts), ctypes.byref(self._cfg),
                                   ctypes.c_int(int(want_jacobians)), ctypes.c_int(threads),
                                   _dp(out))
        return out

    def assemble(self, recs):
        """Fixed edge-order dense assembly (solver.py:428-449)."""
        total = 0.0
        for r in recs:
            total += r[90]
        count = int(sum(int(r[91]) for r in recs))
        free = [p for p in range(self.n_poses) if p != self.gauge]
        slot = {k: 6 * s for s, k in enumerate(free)}
        dim = 6 * (self.n_poses - 1)
        h = np.zeros((dim, dim))
        b = np.zeros(dim)
        iu = np.triu_indices(6)
        for (i, j, *_), r in zip(self.pairs, recs):
            hii = np.zeros((6, 6)); hii[iu] = r[0:21]; hii = hii + np.triu(hii, 1).T
            hjj = np.zeros((6, 6)); hjj[iu] = r[21:42]; hjj = hjj + np.triu(hjj, 1).T
            hij = r[42:78].reshape(6, 6)
            si, sj = slot.get(i), slot.get(j)
            if si is not None:
                h[si:si + 6, si:si + 6] += hii
                b[si:si + 6] += r[78:84]
            if sj is not None:
                h[sj:sj + 6, sj:sj + 6] += hjj
                b[sj:sj + 6] += r[84:90]
            if si is not None and sj is not None:
                h[si:si + 6, sj:sj + 6] += hij
                h[sj:sj + 6, si:si + 6] += hij.T
        return total, count, h, b

    def evaluate(self, pose_arr, want_jacobians=True, threads=None):
        recs = self.records(pose_arr, want_jacobians, threads)
        total, count, h, b = self.assemble(recs)
        if not want_jacobians:
            return total, count, None, None
        return total, count, h, b

    def apply_step(self, pose_arr, gens, delta):
        return apply_step(pose_arr, gens, delta, self.gauge)


def apply_step(pose_arr, gens, delta, gauge):
    """_LevelProblem.apply_step (solver.py:451-460): boxplus every non-gauge pose."""
    out = pose_arr.copy()
    g_out = gens.copy()
    s = 0
    for k in range(pose_arr.shape[0]):
        if k == gauge:
            continue
        R = pose_arr[k, :9].reshape(3, 3)
        t = pose_arr[k, 9:]
        R2, t2, g2 = boxplus(R, t, int(gens[k]), delta[s:s + 6])
        out[k, :9] = R2.reshape(9)
        out[k, 9:] = t2
        g_out[k] = g2
        s += 6
    return out, g_out


@dataclass
class OracleRecord:
    level: int
    iteration: int
    lam: float
    error: float
    valid_blocks: int
    accepted: bool


class OracleUnderConstrained(RuntimeError):
    pass


def solve_level_multi(lp: OracleLevel, pose_arr, gens, level, cfg, max_iterations, threads=None):
    """_solve_level_multi restated (solver.py:495-538)."""
    records = []
    cost, count, h, b = lp.evaluate(pose_arr, True, threads)
    lam = cfg.lm_initial_lambda
    for iteration in range(1, max_iterations + 1):
        if cost <= _COST_FLOOR_PER_BLOCK * max(count, 1):
            break
        damped = h + lam * np.diag(np.diag(h))
        try:
            delta = np.linalg.solve(damped, -b)
        except np.linalg.LinAlgError:
            if iteration == 1:
                raise OracleUnderConstrained("normal equations are singular") from None
            lam *= cfg.lm_factor
            records.append(OracleRecord(level, iteration, lam, cost, count, False))
            if lam > _LAMBDA_CEILING:
                break
            continue
        cand, cgens = lp.apply_step(pose_arr, gens, delta)
        new_cost, new_count, new_h, new_b = lp.evaluate(cand, True, threads)
        rel_change = abs(cost - new_cost) / max(cost, 1e-300)
        if new_cost < cost and new_count > 0:
            pose_arr, gens, cost, count, h, b = cand, cgens, new_cost, new_count, new_h, new_b
            lam = max(lam * 0.5, 1e-12)
            accepted = True
        else:
            lam *= cfg.lm_factor
            accepted = False
        records.append(OracleRecord(level, iteration, lam, cost, count, accepted))
        if rel_change < cfg.termination_rel_decrease or lam > _LAMBDA_CEILING:
            break
    return pose_arr, gens, records


def level_caps(cfg, n_levels):
    caps = list(cfg.max_iterations_per_level)
    while len(caps) < n_levels:
        caps.append(caps[-1])
    return caps[:n_levels]


def hierarchical(problems, cfg, initial=None, levels=None, threads=None):
    """_hierarchical restated (solver.py:585-606); returns (poses (N,12), records)."""
    n_levels = len(problems[0].graph.nodes[0].pyramid)
    schedule = list(range(n_levels)) if levels is None else list(levels)
    poses = initial if initial is not None else [n.pose_guess for n in problems[0].graph.nodes]
    pose_arr, gens = pose_arrays(poses)
    caps = level_caps(cfg, len(schedule))
    records = []
    cache = {}
    for pos, level in enumerate(schedule):
        lp = OracleLevel(problems, level, cfg, cache)
        pose_arr, gens, recs = solve_level_multi(lp, pose_arr, gens, level, cfg, caps[pos], threads)
        records.extend(recs)
    return pose_arr, records


def total_error(problem, poses, level, cfg, suppress_occlusions=True, threads=None):
    lp = OracleLevel([problem], level, cfg)
    if not suppress_occlusions:
        lp.with_tolerance(math.inf)
    pose_arr, _ = pose_arrays(poses)
    cost, count, _, _ = lp.evaluate(pose_arr, False, threads)
    return cost, count


def timed_gn_iteration(lp: OracleLevel, pose_arr, gens, lam, threads=None, pair_subset=None):
    """One GN/LM iteration on the CPU (linearize + solve + update), for the
    bench's CPU baseline: returns (seconds_linearize, seconds_solve_update)."""
    t0 = time.perf_counter()
    recs = lp.records(pose_arr, True, threads, pair_subset)
    t1 = time.perf_counter()
    return recs, t1 - t0
