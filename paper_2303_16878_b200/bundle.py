"""Photometric bundle adjustment: the drop-in entry points.

Same names, arguments, results and errors as the reference solver module
(pkg/src/photoba/solver.py): `SolverConfig` (:56-91), `BAProblem` (:94-103),
`IterationRecord` (:106-122), `SolveResult` (:125-140), `solve_level`
(:555-567), `solve_hierarchical` (:609-616), `solve_fusion` (:619-652),
`total_error` (:655-670), `reproject` (:154-176), `check_connectivity` (:463-486) and the
`UnderConstrainedError` / `FusionConfigError` exceptions.

The Levenberg-Marquardt control flow of `_solve_level_multi`
(solver.py:495-538) is kept verbatim on the host; everything it drives —
linearisation, assembly, the damped solve and the pose update — runs on the
GPU through `device.DeviceLevel` (or its multi-GPU wrapper in
`distributed.py`), with one scalar readback per iteration.  There is no CPU
fallback: without a CUDA device and the built library these calls raise.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .pairgraph import MatchGraph
from .camera import SensorExtrinsics
from .se3 import InvalidPerturbationError, Pose, pose_rows


def reproject(uv, depth, x_i: Pose, x_j: Pose, ext: SensorExtrinsics, cam_src, cam_dst):
    """Source pixels with depth -> destination pixels (the reference's public
    `reproject`, solver.py:154-176): (uv_dst, p_bar, valid), p_bar being the
    point in the destination sensor frame and valid the projection test of
    `project`.  The same chain K1 evaluates per pixel — unproject, into the
    platform frame of i, into platform j, into sensor j, project — as host
    numpy for callers outside the solve loop."""
    from .camera import project, unproject

    p = unproject(cam_src, np.asarray(uv, dtype=float), np.asarray(depth, dtype=float))
    r_o, t_o = ext.offset.rotation, ext.offset.translation
    in_i = p @ r_o.T + t_o                                                    # platform i
    rel = in_i @ x_i.rotation.T + (x_i.translation - x_j.translation)
    p_bar = (rel @ x_j.rotation - t_o) @ r_o                                  # sensor j
    uv_dst, valid = project(cam_dst, p_bar)
    return uv_dst, p_bar, valid


class UnderConstrainedError(RuntimeError):
    """Some poses are not connected to the gauge pose by any edge."""


class FusionConfigError(ValueError):
    """The two sensor problems do not describe the same trajectory."""


COUPLED = "coupled"
CONSECUTIVE = "consecutive"

_LAMBDA_CEILING = 1e12         # solver.py:489
_COST_FLOOR_PER_BLOCK = 1e-18  # solver.py:492
N_LM_ERR_UNDERCONSTRAINED, N_LM_ERR_PERTURBATION = 1, 2  # include/pba.h PBA_LM_ERR_*


@dataclass(frozen=True)
class SolverConfig:
    """Robust kernel, damping, termination and sampling controls."""

    huber_delta_intensity: float = 0.1
    huber_delta_depth: float = 0.1
    huber_delta_normal: float = 0.1
    omega_intensity: float = 1.0
    omega_depth: float = 10.0
    omega_normal: tuple = (1.0, 1.0, 1.0)
    lm_initial_lambda: float = 1e-3
    lm_factor: float = 10.0
    max_iterations_per_level: tuple = (10, 5, 3)
    termination_rel_decrease: float = 1e-4
    occlusion_depth_tolerance: float = 0.05
    pixel_stride: int = 1
    threads: int = 1  # accepted for API compatibility; the GPU path ignores it
    # B200 extension (App. C c3): "cholesky" solves the damped system exactly
    # like the reference's np.linalg.solve; "pcg" uses block-Jacobi PCG to
    # ||r|| <= pcg_tolerance * ||b|| (or pcg_max_iterations, an inexact step).
    linear_solver: str = "cholesky"
    pcg_max_iterations: int = 2000
    pcg_tolerance: float = 1e-12

    def __post_init__(self) -> None:
        positive = (self.huber_delta_intensity, self.huber_delta_depth, self.huber_delta_normal,
                    self.omega_intensity, self.omega_depth, *self.omega_normal)
        if min(positive) <= 0.0:
            raise ValueError("Huber thresholds and information weights must be positive")
        if not 0.0 < self.termination_rel_decrease < 1.0:
            raise ValueError("termination_rel_decrease must lie in (0, 1)")
        if self.pixel_stride < 1 or min(self.max_iterations_per_level) < 1:
            raise ValueError("strides and iteration caps must be >= 1")
        if self.linear_solver not in ("cholesky", "pcg"):
            raise ValueError("linear_solver must be 'cholesky' or 'pcg'")
        if self.pcg_max_iterations < 1 or not self.pcg_tolerance >= 0.0:
            raise ValueError("pcg_max_iterations must be >= 1 and pcg_tolerance >= 0")

    def omega_diagonal(self) -> np.ndarray:
        return np.array([self.omega_intensity, self.omega_depth, *self.omega_normal], dtype=float)


@dataclass
class BAProblem:
    """One sensor's match graph, its mounting offsets and the gauge pose."""

    graph: MatchGraph
    extrinsics: dict = field(default_factory=dict)
    gauge_index: int = 0

    def extrinsics_of(self, sensor_id: str) -> SensorExtrinsics:
        ext = self.extrinsics.get(sensor_id)
        return ext if ext is not None else SensorExtrinsics.identity()


@dataclass
class IterationRecord:
    """One LM iteration, after the accept/reject decision."""

    level: int
    iteration: int
    lam: float
    error: float
    valid_blocks: int
    accepted: bool

    def format_line(self) -> str:
        return (f"level={self.level} iter={self.iteration} lambda={self.lam:.3e} "
                f"error={self.error:.9e} blocks={self.valid_blocks} "
                f"accepted={int(self.accepted)}")


@dataclass
class SolveResult:
    poses: list
    records: list
    level_indices: list
    level_times: list = field(default_factory=list)

    def iterations_per_level(self) -> dict:
        out: dict = {}
        for r in self.records:
            out[r.level] = out.get(r.level, 0) + 1
        return out

    def final_error(self) -> float:
        return self.records[-1].error if self.records else float("nan")


def check_connectivity(problems) -> None:
    """Every pose must reach the gauge through edges of some problem."""
    n = len(problems[0].graph.nodes)
    root = list(range(n))

    def find(a):
        while root[a] != a:
            root[a] = root[root[a]]
            a = root[a]
        return a

    for problem in problems:
        pos = {node.id: k for k, node in enumerate(problem.graph.nodes)}
        for e in problem.graph.edges:
            a, b = find(pos[e.i]), find(pos[e.j])
            if a != b:
                root[a] = b
    g = find(problems[0].gauge_index)
    stranded = [k for k in range(n) if find(k) != g]
    if stranded:
        raise UnderConstrainedError(
            f"poses {stranded} are not connected to gauge pose "
            f"{problems[0].gauge_index}; the problem is under-constrained")


def _level_caps(cfg: SolverConfig, n: int) -> list:
    caps = list(cfg.max_iterations_per_level)
    caps += [caps[-1]] * max(0, n - len(caps))
    return caps[:n]


def _shared_level_count(problems) -> int:
    counts = {len(node.pyramid) for p in problems for node in p.graph.nodes}
    if len(counts) != 1:
        raise ValueError(f"pyramids must share their level count, found {sorted(counts)}")
    return counts.pop()


# ---------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------
class _Runtime:
    """Device + frame store for one solve call (single GPU or one rank)."""

    def __init__(self, device=None):
        import torch

        from . import distributed
        from .device import FrameStore

        if not torch.cuda.is_available():
            raise RuntimeError("paper_2303_16878_b200 needs a CUDA device (no CPU fallback)")
        self.group = distributed.current_group()
        if device is None:
            device = distributed.default_device(self.group)
        self.device = torch.device(device)
        torch.cuda.set_device(self.device)
        self.store = FrameStore(self.device)

    def level(self, problems, level, cfg, tolerance_override=None, need_solver=True):
        """The level backend; need_solver=False (the cost-only path) skips the
        assembly plan and the dense H / Cholesky buffers (O(N^2) memory)."""
        from . import distributed

        return distributed.make_level(problems, level, cfg, self.store, self.group,
                                      tolerance_override=tolerance_override,
                                      need_solver=need_solver)


def _lm_level(backend, level: int, cfg: SolverConfig, max_iterations: int):
    """_solve_level_multi (solver.py:505-537) over a device backend."""
    records = []
    cost, count = backend.evaluate_current()
    lam = cfg.lm_initial_lambda
    device_loop = getattr(backend, "lm_level_device", None)
    if device_loop is not None and max_iterations >= 1 and not (
            cost <= _COST_FLOOR_PER_BLOCK * max(count, 1)):
        # the same loop as below, run on the GPU as one conditional-graph launch
        out = device_loop(cost, count, lam, cfg, max_iterations)
        if out is not None:
            recs, error, _, _ = out
            if error == N_LM_ERR_UNDERCONSTRAINED:
                raise UnderConstrainedError(
                    "normal equations are singular; some pose has no valid observations")
            if error == N_LM_ERR_PERTURBATION:
                raise InvalidPerturbationError(
                    "LM step has ||dq|| >= 1 for some pose; not a quaternion imaginary part")
            return [IterationRecord(level, k + 1, r_lam, r_cost, r_count, acc)
                    for k, (r_lam, r_cost, r_count, acc) in enumerate(recs)]
    for iteration in range(1, max_iterations + 1):
        if cost <= _COST_FLOOR_PER_BLOCK * max(count, 1):
            break
        solve_ok, step_ok, new_cost, new_count = backend.try_step(lam)
        if not solve_ok:
            if iteration == 1:
                raise UnderConstrainedError(
                    "normal equations are singular; some pose has no valid observations")
            lam *= cfg.lm_factor
            records.append(IterationRecord(level, iteration, lam, cost, count, False))
            if lam > _LAMBDA_CEILING:
                break
            continue
        if not step_ok:
            raise InvalidPerturbationError(
                "LM step has ||dq|| >= 1 for some pose; not a quaternion imaginary part")
        rel_change = abs(cost - new_cost) / max(cost, 1e-300)
        if new_cost < cost and new_count > 0:
            backend.accept()
            cost, count = new_cost, new_count
            lam = max(lam * 0.5, 1e-12)
            accepted = True
        else:
            lam *= cfg.lm_factor
            accepted = False
        records.append(IterationRecord(level, iteration, lam, cost, count, accepted))
        if rel_change < cfg.termination_rel_decrease or lam > _LAMBDA_CEILING:
            break
    return records


def _rows_to_poses(rows, gens) -> list:
    return [Pose.from_row(rows[k], int(gens[k])) for k in range(rows.shape[0])]


def _hierarchical(problems, cfg, initial, levels, runtime=None) -> SolveResult:
    check_connectivity(problems)
    n_levels = _shared_level_count(problems)
    schedule = list(range(n_levels)) if levels is None else list(levels)
    if not schedule or any(not 0 <= k < n_levels for k in schedule):
        raise ValueError(f"invalid level schedule {schedule} for {n_levels} levels")
    poses = list(initial) if initial is not None else [n.pose_guess for n in problems[0].graph.nodes]
    rows, gens = pose_rows(poses)
    caps = _level_caps(cfg, len(schedule))
    rt = runtime or _Runtime()
    records, level_times = [], []
    for pos, level in enumerate(schedule):
        t0 = time.perf_counter()
        backend = None  # free the previous level's solver buffers before allocating the next
        backend = rt.level(problems, level, cfg)
        backend.set_poses(rows, gens)
        records.extend(_lm_level(backend, level, cfg, caps[pos]))
        rows, gens = backend.current_rows()
        level_times.append((level, time.perf_counter() - t0))
    return SolveResult(_rows_to_poses(rows, gens), records, schedule, level_times)


def solve_level(problem: BAProblem, poses, level: int, cfg: SolverConfig | None = None,
                max_iterations: int | None = None):
    """LM on one pyramid level with the gauge pose held fixed."""
    cfg = cfg or SolverConfig()
    check_connectivity([problem])
    cap = max_iterations or _level_caps(cfg, level + 1)[level]
    rt = _Runtime()
    backend = rt.level([problem], level, cfg)
    rows, gens = pose_rows(poses)
    backend.set_poses(rows, gens)
    records = _lm_level(backend, level, cfg, cap)
    rows, gens = backend.current_rows()
    return _rows_to_poses(rows, gens), records


def solve_hierarchical(problem: BAProblem, cfg: SolverConfig | None = None, initial=None,
                       levels=None) -> SolveResult:
    """Coarse-to-fine solve, threading the poses through the levels."""
    return _hierarchical([problem], cfg or SolverConfig(), initial, levels)


def solve_fusion(problem_a: BAProblem, problem_b: BAProblem, mode: str = COUPLED,
                 cfg: SolverConfig | None = None, initial=None, levels=None) -> SolveResult:
    """Two-sensor refinement of one platform trajectory (solver.py:619-652)."""
    cfg = cfg or SolverConfig()
    na, nb = len(problem_a.graph.nodes), len(problem_b.graph.nodes)
    if na != nb:
        raise FusionConfigError(f"trajectory lengths disagree: {na} vs {nb}")
    if problem_a.gauge_index != problem_b.gauge_index:
        raise FusionConfigError("fusion problems must share the gauge pose")
    if mode == COUPLED:
        return _hierarchical([problem_a, problem_b], cfg, initial, levels)
    if mode == CONSECUTIVE:
        rt = _Runtime()
        first = _hierarchical([problem_a], cfg, initial, levels, rt)
        second = _hierarchical([problem_b], cfg, first.poses, levels, rt)
        return SolveResult(second.poses, first.records + second.records, second.level_indices,
                           first.level_times + second.level_times)
    raise ValueError(f"unknown fusion mode {mode!r}")


def total_error(problem: BAProblem, poses=None, level: int = 0, cfg: SolverConfig | None = None,
                suppress_occlusions: bool = True):
    """Robustified objective and valid-block count (cost-only path)."""
    cfg = cfg or SolverConfig()
    if poses is None:
        poses = [n.pose_guess for n in problem.graph.nodes]
    rt = _Runtime()
    backend = rt.level([problem], level, cfg,
                       tolerance_override=None if suppress_occlusions else float("inf"),
                       need_solver=False)
    rows, gens = pose_rows(poses)
    return backend.cost_only(rows)
