"""Multi-GPU execution of the BA level: pair sharding + record gather.

One process per GPU (torch.distributed, NCCL over NVLink on the GPU box;
gloo in the CPU tests).  The edge-ordered pair list of a level is split into
contiguous ranges balanced by source-pixel count; every rank keeps all
frames and poses resident and linearises only its range.  Per LM
evaluation the exchange is:

  rank r: records of its pairs (|E_r| x 92 fp64)  --gather-->  rank 0
  rank 0: fixed-edge-order assembly (identical to the single-GPU order),
          damped solve, pose update
  rank 0 --broadcast--> candidate poses (N x 12 fp64) + scalars

Because each per-pair record is computed by the same kernel with the same
chunking whatever rank owns it, and rank 0 assembles in edge order, the
poses are bit-identical for 1, 2, 4 or 8 GPUs (the reference's
thread-count determinism, test_solver.py:456-477).
A reduce of dense H would depend on the rank count, so it is not used.
"""

from __future__ import annotations

import os

import numpy as np
import torch

try:
    import torch.distributed as dist
except Exception:  # pragma: no cover
    dist = None


def current_group():
    """The default process group when more than one rank shares the level
    (PBA_FORCE_SHARDED=1 keeps the sharded path at world size 1, to exercise
    the NCCL collectives on a single-GPU box)."""
    if dist is None or not dist.is_available() or not dist.is_initialized():
        return None
    if dist.get_world_size() == 1 and os.environ.get("PBA_FORCE_SHARDED") != "1":
        return None
    return dist.group.WORLD


def default_device(group):
    if group is None:
        return torch.device("cuda", torch.cuda.current_device())
    local = int(os.environ.get("LOCAL_RANK", dist.get_rank() % max(1, torch.cuda.device_count())))
    return torch.device("cuda", local)


def shard_ranges(pixels_per_pair, world: int) -> list:
    """Contiguous [lo, hi) ranges of the edge list with balanced pixel sums."""
    px = np.asarray(pixels_per_pair, dtype=np.int64)
    n = len(px)
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * max(0, world - 1)
    cum = np.concatenate([[0], np.cumsum(px)])
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        k = int(np.searchsorted(cum, target, side="left"))
        if k > 0 and (target - cum[k - 1]) <= (cum[min(k, n)] - target):
            k -= 1  # nearest boundary, ties to the lower one
        k = min(max(k, bounds[-1]), n)
        bounds.append(k)
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


class ShardedLevel:
    """LM backend over `world` ranks; same interface as DeviceLevel.

    `local` linearises this rank's pairs (`linearize(poses) -> (n_local, 92)`)
    and owns `poses[2]`, `gens[2]`, `cur`; on rank 0 it must also provide the
    solver side (`assemble`, `solve`, `apply_step`, `totals`, status
    pointers).  The collectives run on tensors of `local.device`.
    """

    def __init__(self, local, group, ranges):
        self.local = local
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.ranges = ranges
        self.max_local = max(1, max(hi - lo for lo, hi in ranges))
        dev = local.device
        self._send = torch.zeros((self.max_local, 92), dtype=torch.float64, device=dev)
        # receive buffer on rank 0 only (the other ranks never read records)
        self._gather = torch.zeros((self.world * self.max_local if self.rank == 0 else 1, 92),
                                   dtype=torch.float64, device=dev)
        self._full = torch.zeros((max(1, ranges[-1][1]) if self.rank == 0 else 1, 92),
                                 dtype=torch.float64, device=dev)

    # -- helpers ---------------------------------------------------------------
    def _gather_records(self, recs: torch.Tensor) -> torch.Tensor:
        """Records of every shard to rank 0 only (dist.gather: each rank
        sends max_local x 92 doubles, only rank 0 receives), then placed in
        edge order on rank 0."""
        n = recs.shape[0]
        if n:
            self._send[:n].copy_(recs)
        if n < self.max_local:
            self._send[n:].zero_()
        parts = (list(self._gather.view(self.world, self.max_local, 92).unbind(0))
                 if self.rank == 0 else None)
        dist.gather(self._send, parts, dst=0, group=self.group)
        if self.rank != 0:
            return self._full
        for r, (lo, hi) in enumerate(self.ranges):
            if hi > lo:
                base = r * self.max_local
                self._full[lo:hi].copy_(self._gather[base:base + hi - lo])
        return self._full[: self.ranges[-1][1]]

    def _bcast_scalars(self) -> tuple:
        dist.broadcast(self.local._scal, src=0, group=self.group)
        return self.local._read_scalars()

    # -- backend interface ---------------------------------------------------
    def set_poses(self, rows, gens):
        self.local.set_poses(rows, gens)

    def evaluate_current(self):
        L = self.local
        recs = L.linearize(L.poses[L.cur])
        full = self._gather_records(recs)
        if self.rank == 0:
            L.assemble(full, L.cur)
            L._scal[0:2].copy_(L.totals[L.cur])
        vals, _ = self._bcast_scalars()
        return float(vals[0]), int(round(vals[1]))

    def try_step(self, lam):
        L = self.local
        cur, cand = L.cur, 1 - L.cur
        if self.rank == 0:
            L.solve(cur, lam, L._status_solve_ptr)
            L.apply_step(cur, cand, L._status_step_ptr)
        dist.broadcast(L.poses[cand], src=0, group=self.group)
        dist.broadcast(L.gens[cand], src=0, group=self.group)
        recs = L.linearize(L.poses[cand])
        full = self._gather_records(recs)
        if self.rank == 0:
            L.assemble(full, cand)
            L._scal[0:2].copy_(L.totals[cand])
        vals, ints = self._bcast_scalars()
        return ints[4] == 0, ints[6] == 0, float(vals[0]), int(round(vals[1]))

    def accept(self):
        self.local.accept()

    def current_rows(self):
        return self.local.current_rows()

    def cost_only(self, rows):
        L = self.local
        poses = torch.from_numpy(np.ascontiguousarray(rows, dtype=np.float64)).to(L.device)
        recs = L.linearize(poses, want_jacobians=False)
        full = self._gather_records(recs)
        if self.rank == 0:
            L.sum_totals(full, L._scal[0:2])
        vals, _ = self._bcast_scalars()
        return float(vals[0]), int(round(vals[1]))


def pair_pixels(problems, level, cfg) -> list:
    """Strided source-grid pixels of every pair of the level, in pair order."""
    from .device import LevelTables

    s = int(cfg.pixel_stride)
    tabs = LevelTables(problems, level, cfg)
    out = [0] * len(tabs)
    for p, problem in enumerate(problems):
        px = [-(-n.pyramid.levels[level].intrinsics.width // s)
              * -(-n.pyramid.levels[level].intrinsics.height // s) for n in problem.graph.nodes]
        for k in np.nonzero(tabs.prob == p)[0]:
            out[k] = px[tabs.pose_i[k]]
    return out


def make_level(problems, level, cfg, store, group, tolerance_override=None, need_solver=True):
    """Single-GPU DeviceLevel, or a ShardedLevel over the process group.
    need_solver=False builds no assembly plan / solve buffers (cost-only)."""
    from .device import DeviceLevel

    if group is None:
        return DeviceLevel(problems, level, cfg, store, assemble=need_solver,
                           tolerance_override=tolerance_override)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ranges = shard_ranges(pair_pixels(problems, level, cfg), world)
    local = DeviceLevel(problems, level, cfg, store, pair_range=ranges[rank],
                        assemble=(rank == 0 and need_solver),
                        tolerance_override=tolerance_override)
    return ShardedLevel(local, group, ranges)
