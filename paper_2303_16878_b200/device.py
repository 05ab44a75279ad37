"""GPU-resident state of the BA hot path and the calls into libpba_b200.

`FrameStore` keeps every (frame, level) cue image resident in HBM as the
texel-plane layout (8 planes of 16-byte pairs) plus a mask plane (built on the device from the
reference CueImage channels, csrc/texels.cu).  `DeviceLevel` is the
device replacement of the reference `_LevelProblem` (solver.py:393-460):
pair table, chunk plan, assembly plan, and the buffers of one LM level, with
the linearise / assemble / solve / update steps all enqueued on one CUDA
stream.  Per LM iteration exactly one 64-byte device->host copy happens
(cost, count and the two status words).

torch is used only to own device memory and to name the stream.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import torch

from . import native as N
from .camera import PINHOLE, ray_table

PIXELS_PER_CHUNK_UNIT = 256  # chunk sizes are multiples of this
MAX_CHUNK_UNITS = 32         # <= 8192 pixels per chunk: 64 per thread of K1's 128-thread CTA
SM_COUNT = 148
K1_CTAS_PER_SM = 3           # resident K1 CTAs per SM (168 registers x 128 threads)
LAMBDA_CEILING = 1e12         # solver.py:489 (bundle._LAMBDA_CEILING)
COST_FLOOR_PER_BLOCK = 1e-18  # solver.py:492 (bundle._COST_FLOOR_PER_BLOCK)


def camera_struct(intr) -> N.Camera:
    return N.Camera(N.PBA_PINHOLE if intr.model == PINHOLE else N.PBA_SPHERICAL,
                    int(intr.width), int(intr.height), 0, float(intr.fx), float(intr.fy),
                    float(intr.cx), float(intr.cy), float(intr.depth_min), float(intr.depth_max))


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _struct_tensor(arr, device) -> torch.Tensor:
    raw = bytes(memoryview(arr).cast("B")) if len(arr) else b"\0" * 8
    return torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(device)


def chunk_pixels_for(total_pixels: int) -> int:
    """Source pixels per K1 CTA (chunk).  Chosen from the whole level problem
    (never from a shard) so per-pair sums are identical for any GPU count.
    In multiples of 256 pixels: ~32 waves of resident K1 CTAs (3 per SM on
    148 SMs) so the last wave's tail stays small, between 1,024 and 8,192
    pixels (8,192 = 64 pixels per thread of the 128-thread CTA, the measured
    optimum on c4; c2, 47 M pixels: 3,328 -> 3.23 ms per linearisation vs
    8,192 -> 3.31 / 3.45 ms row-major / tiled); a problem too small for one
    wave at 1,024 gets one wave (DESIGN.md §3 K1).  pba_plan_chunks may round
    a pair's chunk to whole 8-row bands (pair_chunk_pixels)."""
    wave = PIXELS_PER_CHUNK_UNIT * SM_COUNT * K1_CTAS_PER_SM
    units = max(4, min(MAX_CHUNK_UNITS, total_pixels // (wave * 32)))
    if total_pixels < wave * units:  # not even one wave: one wave of smaller chunks
        units = max(1, total_pixels // wave)
    if os.environ.get("PBA_CHUNK_UNITS"):  # (experiments: a fixed chunk size)
        units = max(1, int(os.environ["PBA_CHUNK_UNITS"]))
    return PIXELS_PER_CHUNK_UNIT * units


def block_rows(slot_of_pose, pose_i, pose_j):
    """Block-row CSR (row_ptr, cols) of the damped normal matrix's non-zero
    6x6 blocks: the diagonal plus one block per pair of free poses that share
    an edge, columns ascending (the PCG mat-vec order)."""
    n_free = int((slot_of_pose >= 0).sum())
    si = slot_of_pose[pose_i]
    sj = slot_of_pose[pose_j]
    both = (si >= 0) & (sj >= 0)
    r = np.concatenate([np.arange(n_free), si[both], sj[both]]).astype(np.int64)
    c = np.concatenate([np.arange(n_free), sj[both], si[both]]).astype(np.int64)
    key = np.unique(r * max(1, n_free) + c)
    rows, cols = key // max(1, n_free), key % max(1, n_free)
    row_ptr = np.zeros(n_free + 1, dtype=np.int32)
    np.add.at(row_ptr, rows + 1, 1)
    return np.cumsum(row_ptr).astype(np.int32), cols.astype(np.int32)


def order_chunks(chunk_tab, n_chunks, chunk_pixels, src_of_pair, dst_of_pair,
                 pinhole_of_pair=None):
    """Launch order of the linearisation CTAs.  Results do not depend on it:
    a CTA's partials are stored at its chunk's slot in its pair.

    PBA_CHUNK_ORDER (measured in profiles/r01_chunk_order.json):
      "blk" (default): pairs tiled by (source frame // B, destination frame // B),
            B = 16 for spherical and 32 for pinhole sources (the measured
            optima; PBA_CHUNK_BLOCK overrides both); inside a tile the pairs
            advance chunk position by chunk position, so the CTAs in flight
            read the same row band of ~B source and ~B destination images
            from L2 (c4/200 34.6 -> 32.1 ms, full c3 linearisation 113.4 ->
            101.7 ms);
      "dst": pairs sharing a destination frame interleaved chunk by chunk;
      "src": the same for the source frame;  "pair": edge order.
    """

    order = os.environ.get("PBA_CHUNK_ORDER", "blk")
    if order == "pair" or n_chunks == 0:
        return chunk_tab
    tab = chunk_tab[: 2 * n_chunks].reshape(-1, 2)
    pair = tab[:, 0].astype(np.int64)
    # chunk position inside its pair (the plan lists each pair's chunks in
    # order, pairs ascending; chunk sizes differ between pairs)
    pos = np.arange(len(pair), dtype=np.int64) - np.searchsorted(pair, pair, side="left")
    src = np.asarray(src_of_pair, np.int64)[pair]
    dst = np.asarray(dst_of_pair, np.int64)[pair]
    if order == "blk":
        pin = (np.zeros(len(src_of_pair), np.int64) if pinhole_of_pair is None
               else np.asarray(pinhole_of_pair, np.int64))[pair]
        env = os.environ.get("PBA_CHUNK_BLOCK")
        blk = (np.full(pair.shape, max(1, int(env)), np.int64) if env
               else np.where(pin == 1, 32, 16))
        perm = np.lexsort((pair, pos, dst // blk, src // blk, pin))
    elif order in ("dst", "src"):
        perm = np.lexsort((pair, pos, dst if order == "dst" else src))
    else:
        raise ValueError(f"PBA_CHUNK_ORDER={order!r}: expected blk, dst, src or pair")
    return np.ascontiguousarray(tab[perm].reshape(-1), dtype=np.int32)


def bsr_positions(row_ptr, cols, off_rc):
    """CSR positions of every diagonal block (s, s) and of both orientations
    (r, c) / (c, r) of every off-diagonal assembly target (off_rc pairs).
    The CSR is sorted by (row, column), so one searchsorted on r * n + c."""
    n = len(row_ptr) - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(np.asarray(row_ptr, np.int64)))
    keys = rows * max(n, 1) + np.asarray(cols, np.int64)

    def pos(r, c):
        want = r * max(n, 1) + c
        k = np.searchsorted(keys, want)
        if len(want) and not (np.all(k < len(keys)) and np.array_equal(keys[np.minimum(
                k, len(keys) - 1)], want)):
            raise ValueError("assembly target missing from the block CSR")
        return k.astype(np.int32)

    s = np.arange(n, dtype=np.int64)
    diag = pos(s, s)
    rc = np.asarray(off_rc, dtype=np.int64).reshape(-1, 2)
    off = np.stack([pos(rc[:, 0], rc[:, 1]), pos(rc[:, 1], rc[:, 0])], axis=1).reshape(-1)
    return diag, off.astype(np.int32)


def tile_envelope(slot_of_pose, pose_i, pose_j, dim, tile=64) -> np.ndarray:
    """First possibly non-zero 64-wide tile column of every tile row of the
    damped normal matrix: the envelope of its block sparsity (diagonal
    blocks + one off-diagonal block per pair of free poses).  Cholesky
    fill-in stays inside it, so the solver never touches the rest."""
    n_free = int((slot_of_pose >= 0).sum())
    first = np.arange(n_free, dtype=np.int64)  # first non-zero block column per block row
    si = slot_of_pose[pose_i]
    sj = slot_of_pose[pose_j]
    both = (si >= 0) & (sj >= 0)
    lo = np.minimum(si[both], sj[both])
    hi = np.maximum(si[both], sj[both])
    np.minimum.at(first, hi, lo)
    T = (dim + tile - 1) // tile
    env = np.arange(T, dtype=np.int32)
    rows = np.arange(dim)
    first_col = 6 * first[rows // 6]
    np.minimum.at(env, rows // tile, (first_col // tile).astype(np.int32))
    return np.ascontiguousarray(env, dtype=np.int32)


class FrameStore:
    """Device-resident texel images, one per cue image object."""

    def __init__(self, device):
        self.device = torch.device(device)
        self._frames: dict[int, tuple] = {}
        self._rays: dict[tuple, torch.Tensor] = {}
        self._scratch: torch.Tensor | None = None
        self._lib = N.load()

    def ray(self, intr) -> torch.Tensor:
        key = (intr.model, intr.width, intr.height, intr.fx, intr.fy, intr.cx, intr.cy)
        t = self._rays.get(key)
        if t is None:
            t = torch.from_numpy(ray_table(intr)).to(self.device)
            self._rays[key] = t
        return t

    def _channels(self, cue):
        dev = getattr(cue, "device_intensity", None)
        if dev is not None:
            return (cue.device_intensity.to(self.device, torch.float64).contiguous(),
                    cue.device_depth.to(self.device, torch.float64).contiguous(),
                    cue.device_normals.to(self.device, torch.float64).contiguous())
        out = []
        for a in (cue.intensity, cue.depth, cue.normals):
            h = torch.from_numpy(np.array(a, dtype=np.float64, copy=True))
            out.append(h.to(self.device, non_blocking=False))
        return tuple(out)

    def prefetch(self, cues) -> None:
        """Upload every not-yet-resident cue image of a level at once: one
        texel slab and one mask slab per image size (one allocation each
        instead of two per frame), then the per-frame texel build."""
        todo, seen = {}, set()
        for cue in cues:
            if id(cue) in self._frames or id(cue) in seen:
                continue
            seen.add(id(cue))
            intr = cue.intrinsics
            todo.setdefault((int(intr.height), int(intr.width)), []).append(cue)
        tb = int(self._lib.pba_texel_bytes())
        for (h, w), group in todo.items():
            tex = torch.empty((len(group), h * w * tb), dtype=torch.uint8, device=self.device)
            msk = torch.empty((len(group), h * w), dtype=torch.uint8, device=self.device)
            k = 0
            while k < len(group):
                n = self._batch_run(group, k, h * w)
                if n > 1:  # consecutive frames of one device batch: one batched texel build
                    self._frames_batch(group[k:k + n], tex[k:k + n], msk[k:k + n])
                else:
                    self.frame(group[k], tex[k], msk[k])
                k += max(n, 1)

    @staticmethod
    def _batch_run(group, k, px) -> int:
        """How many cues from group[k] on are consecutive frames of one
        device-resident (n, H, W) batch (device pyramid levels are views
        li[b] of such batches) with identical intrinsics."""
        first = group[k]
        if getattr(first, "device_intensity", None) is None:
            return 1
        chans = ("device_intensity", "device_depth", "device_normals")
        sizes = (px * 8, px * 8, 3 * px * 8)

        def ok(cue):
            return all(getattr(cue, c, None) is not None and getattr(cue, c).dtype == torch.float64
                       and getattr(cue, c).is_contiguous() for c in chans)

        if not ok(first):
            return 1
        base = [getattr(first, c).data_ptr() for c in chans]
        n = 1
        while k + n < len(group):
            cue = group[k + n]
            if (cue.intrinsics != first.intrinsics or not ok(cue)
                    or any(getattr(cue, c).data_ptr() != b + n * sz
                           for c, b, sz in zip(chans, base, sizes))):
                break
            n += 1
        return n

    def _frames_batch(self, cues, texels, mask) -> None:
        """FrameStore.frame for consecutive frames of one device batch through
        pba_build_texels_batch (sub-batches bounded by the scratch size)."""
        first = cues[0]
        intr = first.intrinsics
        cam = camera_struct(intr)
        per = int(self._lib.pba_build_texels_scratch_bytes(ctypes.byref(cam)))
        step = max(1, min(len(cues), (256 << 20) // max(per, 1)))
        if self._scratch is None or self._scratch.numel() < per * step:
            self._scratch = torch.empty(per * step, dtype=torch.uint8, device=self.device)
        ray = self.ray(intr)
        for a in range(0, len(cues), step):
            b = min(len(cues), a + step)
            c0 = cues[a]
            N.check(self._lib.pba_build_texels_batch(
                ctypes.byref(cam), b - a, c0.device_intensity.data_ptr(),
                c0.device_depth.data_ptr(), c0.device_normals.data_ptr(), texels[a].data_ptr(),
                mask[a].data_ptr(), self._scratch.data_ptr(), _stream_ptr(self.device)),
                "pba_build_texels_batch")
            for k in range(a, b):  # keep each cue referenced so its id() stays unique
                self._frames[id(cues[k])] = (cues[k], texels[k], mask[k], ray, camera_struct(intr))

    def frame(self, cue, texels=None, mask=None):
        """(texels, mask, ray table, Camera) of a cue image, uploading on first
        use (into `texels` / `mask` when given, else fresh buffers)."""
        key = id(cue)
        hit = self._frames.get(key)
        if hit is not None:
            return hit[1:]
        intr = cue.intrinsics
        cam = camera_struct(intr)
        h, w = int(intr.height), int(intr.width)
        inten, depth, normals = self._channels(cue)
        if tuple(inten.shape) != (h, w):
            raise ValueError("intrinsics do not match image size")
        if texels is None:
            texels = torch.empty(h * w * int(self._lib.pba_texel_bytes()), dtype=torch.uint8,
                                 device=self.device)
            mask = torch.empty(h * w, dtype=torch.uint8, device=self.device)
        need = int(self._lib.pba_build_texels_scratch_bytes(ctypes.byref(cam)))
        if self._scratch is None or self._scratch.numel() < need:
            self._scratch = torch.empty(need, dtype=torch.uint8, device=self.device)
        N.check(self._lib.pba_build_texels(ctypes.byref(cam), inten.data_ptr(), depth.data_ptr(),
                                           normals.data_ptr(), texels.data_ptr(), mask.data_ptr(),
                                           self._scratch.data_ptr(), _stream_ptr(self.device)),
                "pba_build_texels")
        ray = self.ray(intr)
        # keep `cue` referenced so its id() stays unique while cached
        self._frames[key] = (cue, texels, mask, ray, cam)
        return texels, mask, ray, cam

    def texel_bytes(self) -> int:
        return sum(v[1].numel() + v[2].numel() for v in self._frames.values())


class LevelTables:
    """The contexts of _LevelProblem.__init__ (solver.py:400-414) as arrays,
    in its pair order (problem by problem, edge order): per pair the problem,
    the two node (pose) indices and the occlusion tolerance (solver.py:410);
    cross-sensor edges raise FusionConfigError (solver.py:406-407).  One pass
    over the edges instead of a tuple per pair."""

    def __init__(self, problems, level, cfg, tolerance_override=None):
        self.problems = problems
        prob, pi, pj, tol = [], [], [], []
        for p, problem in enumerate(problems):
            nodes = problem.graph.nodes
            index_of = {n.id: k for k, n in enumerate(nodes)}
            edges = problem.graph.edges
            ei = np.fromiter((index_of[e.i] for e in edges), dtype=np.int64, count=len(edges))
            ej = np.fromiter((index_of[e.j] for e in edges), dtype=np.int64, count=len(edges))
            sensor_code = {}
            codes = np.fromiter((sensor_code.setdefault(n.sensor_id, len(sensor_code))
                                 for n in nodes), dtype=np.int64, count=len(nodes))
            if len(edges) and np.any(codes[ei] != codes[ej]):
                from .bundle import FusionConfigError
                raise FusionConfigError("edges must connect frames of one sensor")
            scale = np.fromiter((n.pyramid.scales[level] for n in nodes), dtype=np.float64,
                                count=len(nodes))
            prob.append(np.full(len(edges), p, dtype=np.int64))
            pi.append(ei)
            pj.append(ej)
            tol.append(cfg.occlusion_depth_tolerance / scale[ei] if tolerance_override is None
                       else np.full(len(edges), float(tolerance_override)))
        cat = (lambda a, dt: np.concatenate(a).astype(dt) if a else np.zeros(0, dt))
        self.prob = cat(prob, np.int64)
        self.pose_i = cat(pi, np.int64)
        self.pose_j = cat(pj, np.int64)
        self.tol = cat(tol, np.float64)

    def __len__(self) -> int:
        return len(self.pose_i)


def config_struct(cfg) -> N.Config:
    c = N.Config()
    c.huber_delta[:] = [cfg.huber_delta_intensity, cfg.huber_delta_depth, cfg.huber_delta_normal]
    c.omega[:] = [cfg.omega_intensity, cfg.omega_depth, *cfg.omega_normal]
    c.pixel_stride = int(cfg.pixel_stride)
    return c


class DeviceLevel:
    """One pyramid level of one (or several, for fusion) BA problems on one GPU.

    `pair_range` restricts the linearisation to a contiguous slice of the
    edge-ordered pair list (the multi-GPU shard); `assemble=True` builds the
    dense-assembly plan and solve buffers (the rank that solves).
    """

    def __init__(self, problems, level, cfg, store: FrameStore, *, pair_range=None,
                 assemble=True, tolerance_override=None):
        self.lib = N.load()
        self.store = store
        self.device = store.device
        self.cfg = cfg
        self.level = level
        self.kernel_events = None  # list -> (start, stop) CUDA events per pba_linearize call
        self.solve_events = None   # same for pba_solve_dense
        self.n_poses = len(problems[0].graph.nodes)
        self.gauge = problems[0].gauge_index
        self.ccfg = config_struct(cfg)
        tabs = LevelTables(problems, level, cfg, tolerance_override)
        self.n_pairs_total = len(tabs)
        self.pose_i = tabs.pose_i.astype(np.int32)
        self.pose_j = tabs.pose_j.astype(np.int32)
        # chunk size from the whole level (shard-independent)
        stride = int(cfg.pixel_stride)
        node_px = [np.fromiter((math.ceil(n.pyramid.levels[level].intrinsics.width / stride)
                                * math.ceil(n.pyramid.levels[level].intrinsics.height / stride)
                                for n in pr.graph.nodes), dtype=np.int64,
                               count=len(pr.graph.nodes)) for pr in problems]
        pair_px = np.zeros(len(tabs), dtype=np.int64)
        for p, px in enumerate(node_px):
            sel = tabs.prob == p
            pair_px[sel] = px[tabs.pose_i[sel]]
        total_px = int(pair_px.sum())
        self.total_pixels = total_px
        self.chunk_pixels = chunk_pixels_for(total_px)
        lo, hi = (0, len(tabs)) if pair_range is None else pair_range
        self.pair_lo, self.pair_hi = lo, hi
        m_prob, m_i, m_j = tabs.prob[lo:hi], tabs.pose_i[lo:hi], tabs.pose_j[lo:hi]
        self.n_pairs = hi - lo
        # frame / extrinsics tables for this shard: one slot per node image
        # used, in first-use order (source then destination, pair by pair)
        order = np.stack([m_i, m_j], axis=1).reshape(-1) if self.n_pairs else np.zeros(0, np.int64)
        order_prob = np.repeat(m_prob, 2)
        key = order_prob * (1 << 32) + order
        _, first = np.unique(key, return_index=True)
        used = key[np.sort(first)]  # unique nodes, first-use order
        used_nodes = [problems[int(k >> 32)].graph.nodes[int(k & 0xFFFFFFFF)] for k in used]
        store.prefetch([n.pyramid.levels[level] for n in used_nodes])
        frames, frame_slot, ext_rows, ext_slot = [], {}, [], {}
        node_slot = np.empty(len(used), dtype=np.int64)
        for u, node in enumerate(used_nodes):
            cue = node.pyramid.levels[level]
            s_ = frame_slot.get(id(cue))
            if s_ is None:
                tex, mask, ray, cam = store.frame(cue)
                s_ = frame_slot[id(cue)] = len(frames)
                frames.append(N.Frame(tex.data_ptr(), mask.data_ptr(), ray.data_ptr(), cam))
            node_slot[u] = s_
        ext_of_sensor: dict = {}

        def ext_index(p, sensor_id):
            e_ = ext_of_sensor.get((p, sensor_id))
            if e_ is None:
                off = problems[p].extrinsics_of(sensor_id).offset
                ekey = (np.asarray(off.rotation, float).tobytes(),
                        np.asarray(off.translation, float).tobytes())
                if ekey not in ext_slot:
                    ext_slot[ekey] = len(ext_rows)
                    ext_rows.append(np.concatenate([np.asarray(off.rotation, float).reshape(9),
                                                    np.asarray(off.translation, float).reshape(3)]))
                e_ = ext_of_sensor[(p, sensor_id)] = ext_slot[ekey]
            return e_

        node_ext = np.array([ext_index(int(k >> 32), n.sensor_id)
                             for k, n in zip(used, used_nodes)], dtype=np.int64)
        idx = np.zeros((max(1, self.n_pairs), 5), dtype=np.int32)  # pose_i, pose_j, src, dst, ext
        tols = np.zeros(max(1, self.n_pairs))
        if self.n_pairs:
            pos_i = np.searchsorted(used, m_prob * (1 << 32) + m_i, sorter=np.argsort(used))
            pos_j = np.searchsorted(used, m_prob * (1 << 32) + m_j, sorter=np.argsort(used))
            srt = np.argsort(used)
            ui, uj = srt[pos_i], srt[pos_j]
            idx[: self.n_pairs] = np.stack([m_i, m_j, node_slot[ui], node_slot[uj], node_ext[ui]],
                                           axis=1).astype(np.int32)
            tols[: self.n_pairs] = tabs.tol[lo:hi]
        # the pba_pair / pba_camera tables built in one go (32 B / 64 B records)
        pair_rec = np.zeros(max(1, self.n_pairs), dtype=[("i", "<i4", 6), ("tol", "<f8")])
        pair_rec["i"][:, :5] = idx
        pair_rec["tol"] = tols
        pairs = (N.Pair * max(1, self.n_pairs)).from_buffer_copy(pair_rec.tobytes())
        cam_bytes = np.frombuffer(b"".join(bytes(f.cam) for f in frames) or bytes(64),
                                  dtype=np.uint8).reshape(-1, ctypes.sizeof(N.Camera))
        src_cams = (N.Camera * max(1, self.n_pairs)).from_buffer_copy(
            cam_bytes[idx[:, 2]].tobytes())
        if self.n_pairs and any(frames[d].cam.model == N.PBA_PINHOLE for d in set(idx[:, 3])):
            self.ccfg.flags |= N.PBA_CFG_PINHOLE_DST
        n_chunks = ctypes.c_int64(0)
        N.check(self.lib.pba_plan_chunks(pairs, self.n_pairs, src_cams, stride, self.chunk_pixels,
                                         None, None, ctypes.byref(n_chunks)), "pba_plan_chunks")
        self.n_chunks = int(n_chunks.value)
        chunk_tab = np.zeros(max(1, 2 * self.n_chunks), dtype=np.int32)
        offsets = np.zeros(self.n_pairs + 1, dtype=np.int32)
        N.check(self.lib.pba_plan_chunks(pairs, self.n_pairs, src_cams, stride, self.chunk_pixels,
                                         chunk_tab.ctypes.data, offsets.ctypes.data,
                                         ctypes.byref(n_chunks)), "pba_plan_chunks")
        frame_pinhole = np.array([int(f.cam.model == N.PBA_PINHOLE) for f in frames] or [0])
        chunk_tab = order_chunks(chunk_tab, self.n_chunks, self.chunk_pixels,
                                 idx[: self.n_pairs, 2], idx[: self.n_pairs, 3],
                                 frame_pinhole[idx[: self.n_pairs, 2]])
        dev = self.device
        self.frames_t = _struct_tensor((N.Frame * max(1, len(frames)))(*frames), dev)
        self.pairs_t = _struct_tensor(pairs, dev)
        self.chunks_t = torch.from_numpy(chunk_tab).to(dev)
        self.offsets_t = torch.from_numpy(offsets).to(dev)
        ext_arr = np.array(ext_rows, dtype=np.float64).reshape(-1, 12)
        self.ext_t = torch.from_numpy(ext_arr if len(ext_arr) else np.zeros((1, 12))).to(dev)
        # chunk partials + one setup per pair (pba_linearize_scratch_bytes)
        self.partials = torch.empty(
            max(16, int(self.lib.pba_linearize_scratch_bytes(self.n_pairs, self.n_chunks))),
            dtype=torch.uint8, device=dev)
        self.records = torch.zeros((max(1, self.n_pairs), N.RECORD_DOUBLES), dtype=torch.float64,
                                   device=dev)
        self.pixels_shard = int(pair_px[lo:hi].sum())
        self._scal = torch.zeros(8, dtype=torch.float64, device=dev)
        self._scal_host = torch.zeros(8, dtype=torch.float64).pin_memory()
        # LM damping read by the solve kernels from device memory, so one
        # captured step (solve -> update -> linearise -> assemble -> readback)
        # replays with a new lambda (CUDA graph per current buffer, try_step)
        self._lam_dev = torch.zeros(1, dtype=torch.float64, device=dev)
        self._lam_host = torch.zeros(1, dtype=torch.float64).pin_memory()
        self._plan_ready = False
        self._graphs = [None, None]
        self._graph_events = [None, None]
        self._eager_steps = [0, 0]
        self._graph_failed = False
        self._capture_lin_events = None
        self._graph_nlaunch = [0, 0]        # library kernels in each captured step
        self._lm_loop = None                # device-resident LM level (lm_level_device)
        self._lm_loop_failed = False
        self._lm_loop_error = None
        self._lm_nlaunch = 0
        self.lm_device_iterations = 0
        self.graph_launches_replayed = 0    # library kernels launched through replays
        self.poses = [torch.zeros((self.n_poses, 12), dtype=torch.float64, device=dev)
                      for _ in range(2)]
        self.gens = [torch.zeros(self.n_poses, dtype=torch.int32, device=dev) for _ in range(2)]
        self.cur = 0
        self.has_solver = False
        if assemble:
            self._build_solver()

    # ---- solver side --------------------------------------------------------
    def _build_solver(self):
        lib, dev = self.lib, self.device
        slot = np.full(self.n_poses, -1, dtype=np.int32)
        s = 0
        for k in range(self.n_poses):
            if k != self.gauge:
                slot[k] = s
                s += 1
        self.n_free = s
        self.dim = 6 * s
        n_off = ctypes.c_int32(0)
        N.check(lib.pba_plan_assembly(slot.ctypes.data, self.n_poses, self.pose_i.ctypes.data,
                                      self.pose_j.ctypes.data, self.n_pairs_total, None, None,
                                      None, None, None, ctypes.byref(n_off)), "pba_plan_assembly")
        self.n_off = int(n_off.value)
        diag_ptr = np.zeros(self.n_free + 1, np.int32)
        diag_items = np.zeros(max(1, 2 * self.n_pairs_total), np.int32)
        off_ptr = np.zeros(self.n_off + 1, np.int32)
        off_rc = np.zeros(max(1, 2 * self.n_off), np.int32)
        off_items = np.zeros(max(1, self.n_pairs_total), np.int32)
        N.check(lib.pba_plan_assembly(slot.ctypes.data, self.n_poses, self.pose_i.ctypes.data,
                                      self.pose_j.ctypes.data, self.n_pairs_total,
                                      diag_ptr.ctypes.data, diag_items.ctypes.data,
                                      off_ptr.ctypes.data, off_rc.ctypes.data,
                                      off_items.ctypes.data, ctypes.byref(n_off)),
                "pba_plan_assembly")
        t = lambda a: torch.from_numpy(a).to(dev)
        self.plan = [t(diag_ptr), t(diag_items), t(off_ptr), t(off_rc), t(off_items)]
        d = max(1, self.dim)
        # block-sparse H (north_star: "into the block-sparse H/b"): the 6x6
        # blocks of the block-row CSR of the damped system, diagonal + both
        # orientations of every off-diagonal block (pba_assemble_bsr)
        row_ptr, cols = block_rows(slot, self.pose_i, self.pose_j)
        self.n_blocks = int(row_ptr[-1])
        diag_blk, off_blk = bsr_positions(row_ptr, cols, off_rc[: 2 * self.n_off])
        self.bsr = [t(row_ptr), t(cols), t(diag_blk), t(off_blk if len(off_blk) else
                                                          np.zeros(2, np.int32))]
        self.Hb = [torch.zeros((max(1, self.n_blocks), 36), dtype=torch.float64, device=dev)
                   for _ in range(2)]
        self.b = [torch.zeros(d, dtype=torch.float64, device=dev) for _ in range(2)]
        self.totals = [torch.zeros(2, dtype=torch.float64, device=dev) for _ in range(2)]
        # getattr: a reference photoba SolverConfig (no B200 fields) is accepted as-is
        self.pcg = getattr(self.cfg, "linear_solver", "cholesky") == "pcg" and self.n_free > 0
        if not self.pcg:  # the Cholesky workspace (D x D) is not needed by PCG
            self.work = torch.empty(max(8, int(lib.pba_solve_work_bytes(d))), dtype=torch.uint8,
                                    device=dev)
        self.delta = torch.zeros(d, dtype=torch.float64, device=dev)
        self.tile_env = tile_envelope(slot, self.pose_i, self.pose_j, self.dim)
        if self.pcg:
            self.pcg_work = torch.empty(max(8, int(lib.pba_pcg_work_bytes(self.n_free))),
                                        dtype=torch.uint8, device=dev)
            self.pcg_info = torch.zeros(3, dtype=torch.float64, device=dev)
        self.has_solver = True

    # ---- primitive steps -----------------------------------------------------
    def linearize(self, poses_t: torch.Tensor, want_jacobians: bool = True) -> torch.Tensor:
        """Per-pair records of this shard at `poses_t` (device (N,12) fp64)."""
        if self.n_pairs == 0:
            return self.records[:0]
        stream = torch.cuda.current_stream(self.device)
        cap = getattr(self, "_capture_lin_events", None)  # graph-owned events while capturing
        ev = self.kernel_events if cap is None else None
        if cap:
            cap[0].record(stream)
        elif ev is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        N.check(self.lib.pba_linearize(
            self.frames_t.data_ptr(), self.pairs_t.data_ptr(), self.n_pairs,
            self.chunks_t.data_ptr(), self.n_chunks, self.offsets_t.data_ptr(), self.chunk_pixels,
            poses_t.data_ptr(), self.ext_t.data_ptr(), ctypes.byref(self.ccfg),
            int(bool(want_jacobians)), self.partials.data_ptr(), self.records.data_ptr(),
            stream.cuda_stream), "pba_linearize")
        if cap:
            cap[1].record(stream)
        elif ev is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(stream)
            ev.append((e0, e1))
        return self.records[: self.n_pairs]

    def assemble(self, records: torch.Tensor, which: int) -> None:
        dp, di, op, orc, oi = self.plan
        _, _, dblk, oblk = self.bsr
        N.check(self.lib.pba_assemble_bsr(
            records.data_ptr(), self.n_pairs_total, self.n_free, dp.data_ptr(), di.data_ptr(),
            self.n_off, op.data_ptr(), oi.data_ptr(), dblk.data_ptr(), oblk.data_ptr(),
            self.Hb[which].data_ptr(), self.b[which].data_ptr(), self.totals[which].data_ptr(),
            _stream_ptr(self.device)), "pba_assemble_bsr")

    def dense_H(self, which: int) -> torch.Tensor:
        """The assembled normal matrix of buffer `which` as a dense (dim, dim)
        tensor (tests and diagnostics; the solver never forms it)."""
        rp, cols, _, _ = (x.cpu().numpy() for x in self.bsr)
        rows = np.repeat(np.arange(self.n_free), np.diff(rp))
        blocks = self.Hb[which][: self.n_blocks].reshape(-1, 6, 6)
        H = torch.zeros((self.n_free, 6, self.n_free, 6), dtype=torch.float64, device=self.device)
        H[torch.from_numpy(rows).to(self.device), :, torch.from_numpy(cols.astype(np.int64))
          .to(self.device), :] = blocks
        return H.reshape(self.dim, self.dim)

    def sum_totals(self, records: torch.Tensor, out: torch.Tensor) -> None:
        N.check(self.lib.pba_sum_totals(records.data_ptr(), records.shape[0], out.data_ptr(),
                                        _stream_ptr(self.device)), "pba_sum_totals")

    def solve(self, which: int, lam, status_ptr: int) -> None:
        """Damped solve of buffer `which`.  lam=None: lambda is read from
        self._lam_dev on the device (the captured-step form)."""
        ev = self.solve_events if getattr(self, "_capture_lin_events", None) is None else None
        if ev is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream(self.device))
        lam_v = 0.0 if lam is None else float(lam)
        lam_p = self._lam_dev.data_ptr() if lam is None else None
        rp, cols, dblk, _ = self.bsr
        if self.pcg:
            N.check(self.lib.pba_solve_pcg_bsr(self.Hb[which].data_ptr(), self.b[which].data_ptr(),
                                               self.n_free, lam_v, lam_p, rp.data_ptr(),
                                               cols.data_ptr(), dblk.data_ptr(),
                                               int(getattr(self.cfg, "pcg_max_iterations", 2000)),
                                               float(getattr(self.cfg, "pcg_tolerance", 1e-12)),
                                               self.pcg_work.data_ptr(), self.delta.data_ptr(),
                                               status_ptr, self.pcg_info.data_ptr(),
                                               _stream_ptr(self.device)), "pba_solve_pcg_bsr")
        else:
            flags = N.PBA_SOLVE_REUSE_PLAN if self._plan_ready else 0
            N.check(self.lib.pba_solve_dense_bsr(self.Hb[which].data_ptr(), rp.data_ptr(),
                                                 cols.data_ptr(), self.b[which].data_ptr(),
                                                 self.dim, lam_v, lam_p, self.tile_env.ctypes.data,
                                                 self.work.data_ptr(), flags,
                                                 self.delta.data_ptr(), status_ptr,
                                                 _stream_ptr(self.device)), "pba_solve_dense_bsr")
            self._plan_ready = True  # the tile tables are now in self.work
        if ev is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(torch.cuda.current_stream(self.device))
            ev.append((e0, e1))

    def apply_step(self, src: int, dst: int, status_ptr: int) -> None:
        N.check(self.lib.pba_apply_step(self.poses[src].data_ptr(), self.gens[src].data_ptr(),
                                        self.delta.data_ptr(), self.n_poses, self.gauge,
                                        self.poses[dst].data_ptr(), self.gens[dst].data_ptr(),
                                        status_ptr, _stream_ptr(self.device)), "pba_apply_step")

    # ---- scalar readback -----------------------------------------------------
    def _read_scalars(self):
        self._scal_host.copy_(self._scal, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        vals = self._scal_host.numpy().copy()
        ints = self._scal_host.view(torch.int32).numpy().copy()
        return vals, ints

    @property
    def _status_solve_ptr(self) -> int:
        return self._scal.data_ptr() + 16

    @property
    def _status_step_ptr(self) -> int:
        return self._scal.data_ptr() + 24

    # ---- single-GPU LM backend (used by bundle._lm_level) --------------------
    def set_poses(self, rows: np.ndarray, gens: np.ndarray) -> None:
        self.cur = 0
        self.poses[0].copy_(torch.from_numpy(np.ascontiguousarray(rows, dtype=np.float64)))
        self.gens[0].copy_(torch.from_numpy(np.ascontiguousarray(gens, dtype=np.int32)))

    def evaluate_current(self):
        """Linearise + assemble at the current poses; returns (cost, count)."""
        recs = self.linearize(self.poses[self.cur])
        self.assemble(recs, self.cur)
        self._scal[0:2].copy_(self.totals[self.cur])
        vals, _ = self._read_scalars()
        return float(vals[0]), int(round(vals[1]))

    def try_step(self, lam: float):
        """solve -> update -> linearise + assemble the candidate, one readback.

        The second and later steps from the same current buffer replay a
        CUDA graph of this whole sequence (lambda in device memory), so a
        small problem's step costs one graph launch instead of ~20 kernel
        launches and their host calls (PBA_GRAPH=0 disables it).

        Returns (solve_ok, step_ok, new_cost, new_count)."""
        cur, cand = self.cur, 1 - self.cur
        if self._graph_enabled():
            g = self._graphs[cur]
            if g is None and self._plan_ready and self._graph_pays(cur):
                g = self._capture_step(cur)
            if g is not None:
                self._lam_host[0] = lam
                g.replay()
                self.graph_launches_replayed += self._graph_nlaunch[cur]
                torch.cuda.current_stream(self.device).synchronize()
                ev = self._graph_events[cur]
                if ev is not None and self.kernel_events is not None:
                    self.kernel_events.append(ev[0].elapsed_time(ev[1]))
                if ev is not None and self.solve_events is not None and self.has_solver:
                    self.solve_events.append(ev[2].elapsed_time(ev[3]))
                vals = self._scal_host.numpy().copy()
                ints = self._scal_host.view(torch.int32).numpy().copy()
                return ints[4] == 0, ints[6] == 0, float(vals[0]), int(round(vals[1]))
        self._eager_steps[cur] += 1
        self._step_body(cur, cand, lam)
        vals, ints = self._read_scalars()
        return ints[4] == 0, ints[6] == 0, float(vals[0]), int(round(vals[1]))

    def _step_body(self, cur: int, cand: int, lam) -> None:
        self.solve(cur, lam, self._status_solve_ptr)
        self.apply_step(cur, cand, self._status_step_ptr)
        recs = self.linearize(self.poses[cand])
        self.assemble(recs, cand)
        self._scal[0:2].copy_(self.totals[cand])

    # ---- CUDA-graph step ------------------------------------------------------
    def _graph_pays(self, cur: int) -> bool:
        """Capture lazily only where a replay saves a visible share of the
        step: a problem small enough that host launch work matters
        (<= 64 M source pixels per linearisation) that has already run two
        eager steps from this buffer (so an LM level that stops after a few
        iterations never pays for a capture).  prepare_graphs() forces it."""
        return self.pixels_shard <= (1 << 26) and self._eager_steps[cur] >= 2

    def prepare_graphs(self) -> None:
        """Capture the step graphs of both buffers now (after one eager step),
        so no capture happens inside a timed loop."""
        if self._graph_enabled() and self._plan_ready:
            for c in (0, 1):
                if self._graphs[c] is None:
                    self._capture_step(c)

    def _graph_enabled(self) -> bool:
        return (self.has_solver and not self._graph_failed
                and os.environ.get("PBA_GRAPH", "1") != "0")

    def _capture_step(self, cur: int):
        """Capture one try_step from buffer `cur` (lambda from pinned host
        memory -> device, solve, update, linearise, assemble, scalars -> pinned
        host memory).  Events around the linearisation and the solve are
        captured too, so the bench can still time the kernels per replay."""
        cand = 1 - cur
        stream = torch.cuda.Stream(self.device)
        stream.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        events = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(4)]
        n0 = int(self.lib.pba_kernel_launches())
        try:
            with torch.cuda.graph(g, stream=stream):
                self._capture_lin_events = (events[0], events[1])
                self._lam_dev.copy_(self._lam_host, non_blocking=True)
                events[2].record()
                self.solve(cur, None, self._status_solve_ptr)
                events[3].record()
                self.apply_step(cur, cand, self._status_step_ptr)
                recs = self.linearize(self.poses[cand])
                self.assemble(recs, cand)
                self._scal[0:2].copy_(self.totals[cand])
                self._scal_host.copy_(self._scal, non_blocking=True)
        except Exception:  # capture unsupported here (e.g. the cooperative PCG launch)
            self._graph_failed = True
            self._capture_lin_events = None
            torch.cuda.synchronize(self.device)
            return None
        self._capture_lin_events = None
        torch.cuda.current_stream(self.device).wait_stream(stream)
        self._graph_nlaunch[cur] = int(self.lib.pba_kernel_launches()) - n0
        self._graphs[cur] = g
        self._graph_events[cur] = events
        return g

    # ---- device-resident LM level (csrc/lmloop.cu) ---------------------------
    LM_RECORD_CAPACITY = 256

    def lm_loop_ready(self) -> bool:
        """Whether lm_level_device runs here (policy + a captured loop graph)."""
        if (os.environ.get("PBA_LM_DEVICE", "1") == "0" or not self._graph_enabled()
                or self.pixels_shard > (1 << 26)):
            return False
        if self.cur != 0:  # the loop body is captured on buffer 0
            for bufs in (self.poses, self.gens, self.Hb, self.b, self.totals):
                bufs[0].copy_(bufs[1])
            self.cur = 0
        return self._lm_loop_graph() is not None

    def lm_level_device(self, cost: float, count: int, lam: float, cfg, max_iterations: int,
                        lam_ceiling: float = LAMBDA_CEILING, details: bool = False,
                        events=None):
        """The iterations of bundle._lm_level (solver.py:505-537) as one graph
        launch: a conditional WHILE node replays solve -> update -> linearise
        -> assemble -> decide (+ copy on accept) until the device-side decision
        stops the loop; the host reads the records once.  Returns
        (records [(lambda, cost, count, accepted)], error code, cost, count),
        or None where the loop graph is not used (large problems, where a
        host round trip per iteration is negligible; PBA_LM_DEVICE=0; a
        backend whose step cannot be captured) — the caller then runs the
        host loop.  `events` (start, stop) are recorded on the stream around
        the loop launch alone (the bench's timed region)."""
        if max_iterations > self.LM_RECORD_CAPACITY or not self.lm_loop_ready():
            return None
        loop = self._lm_loop
        st = self._lm_state_host
        st.zero_()
        st[N.LM_COST], st[N.LM_COUNT], st[N.LM_LAMBDA] = cost, float(count), lam
        st[N.LM_FACTOR] = cfg.lm_factor
        st[N.LM_REL_TOL] = cfg.termination_rel_decrease
        st[N.LM_LAMBDA_CEILING], st[N.LM_COST_FLOOR] = lam_ceiling, COST_FLOOR_PER_BLOCK
        st[N.LM_ITERATION], st[N.LM_MAX_ITERATIONS] = 1.0, float(max_iterations)
        stream = torch.cuda.current_stream(self.device)
        self._lm_state.copy_(st, non_blocking=True)
        self._lam_dev.copy_(self._lm_state[N.LM_LAMBDA:N.LM_LAMBDA + 1])
        if events is not None:
            events[0].record(stream)
        N.check(self.lib.pba_lm_loop_launch(loop, stream.cuda_stream), "pba_lm_loop_launch")
        if events is not None:
            events[1].record(stream)
        st.copy_(self._lm_state, non_blocking=True)
        stream.synchronize()
        n = int(st[N.LM_N_RECORDS])
        recs = self._lm_records[: N.LM_RECORD_DOUBLES * n].cpu().numpy().reshape(
            n, N.LM_RECORD_DOUBLES)
        iters = int(st[N.LM_ITERATION]) - 1
        self.graph_launches_replayed += self._lm_nlaunch * iters
        self.lm_device_iterations += iters
        out = [(float(r[0]), float(r[1]), int(round(r[2])), bool(r[3])) for r in recs]
        if details:  # + the candidate's (cost, count) per iteration
            out = [o + (float(r[4]), int(round(r[5]))) for o, r in zip(out, recs)]
        return (out, int(st[N.LM_ERROR]), float(st[N.LM_COST]),
                int(round(float(st[N.LM_COUNT]))))

    def _lm_loop_graph(self):
        if self._lm_loop is not None or self._lm_loop_failed:
            return self._lm_loop
        if not self._plan_ready:  # the solver's tile tables go up once, outside the capture
            self.solve(0, 1.0, self._status_solve_ptr)
        dev = self.device
        self._lm_state = torch.zeros(N.LM_STATE_DOUBLES, dtype=torch.float64, device=dev)
        self._lm_state_host = torch.zeros(N.LM_STATE_DOUBLES, dtype=torch.float64).pin_memory()
        self._lm_records = torch.zeros(N.LM_RECORD_DOUBLES * self.LM_RECORD_CAPACITY,
                                       dtype=torch.float64, device=dev)
        segs = [(self.poses[0], self.poses[1]), (self.gens[0], self.gens[1]),
                (self.Hb[0], self.Hb[1]), (self.b[0], self.b[1]),
                (self.totals[0], self.totals[1])]
        n = len(segs)
        dst = (ctypes.c_void_p * n)(*[d.data_ptr() for d, _ in segs])
        src = (ctypes.c_void_p * n)(*[s_.data_ptr() for _, s_ in segs])
        nbytes = (ctypes.c_int64 * n)(*[d.numel() * d.element_size() for d, _ in segs])
        stream = torch.cuda.Stream(dev)
        stream.wait_stream(torch.cuda.current_stream(dev))
        torch.cuda.synchronize(dev)
        loop, handle = ctypes.c_void_p(), ctypes.c_uint64()
        # (no event-record nodes: a conditional node's body may not hold them)
        self._lm_events = None
        n0 = int(self.lib.pba_kernel_launches())
        ok = False
        if self.lib.pba_lm_loop_begin(stream.cuda_stream, ctypes.byref(loop),
                                      ctypes.byref(handle)) == N.PBA_OK:
            try:
                stamp = self._lm_stamp_fn(stream)
                with torch.cuda.stream(stream):
                    self._capture_lin_events = ()  # capturing: no per-call timing events
                    stamp(0)
                    self.solve(0, None, self._status_solve_ptr)
                    stamp(1)
                    self.apply_step(0, 1, self._status_step_ptr)
                    stamp(2)
                    recs = self.linearize(self.poses[1])
                    stamp(3)
                    self.assemble(recs, 1)
                    stamp(4)
                    N.check(self.lib.pba_lm_decide(
                        self._lm_state.data_ptr(), self._lm_records.data_ptr(),
                        self._status_solve_ptr, self._status_step_ptr,
                        self.totals[1].data_ptr(), self._lam_dev.data_ptr(), handle.value,
                        dst, src, nbytes, n, stream.cuda_stream), "pba_lm_decide")
                    stamp(5)
                N.check(self.lib.pba_lm_loop_end(loop), "pba_lm_loop_end")
                ok = True
            except Exception as exc:  # capture unsupported here: the host loop runs instead
                self._lm_loop_error = repr(exc)
            finally:
                self._capture_lin_events = None
        if not ok:
            if loop.value:
                self.lib.pba_lm_loop_destroy(loop)
            torch.cuda.synchronize(dev)
            self._lm_loop_failed = True
            return None
        torch.cuda.current_stream(dev).wait_stream(stream)
        self._lm_nlaunch = int(self.lib.pba_kernel_launches()) - n0
        self._lm_loop = loop
        self._lm_loop_handle = handle
        self._lm_stream = stream
        return loop

    def _lm_stamp_fn(self, stream):
        """PBA_LM_STAMPS=1 (diagnostics): globaltimer stamps between the
        phases of the captured loop body into self.lm_stamps (8 per iteration)."""
        if os.environ.get("PBA_LM_STAMPS") != "1":
            return lambda slot: None
        self.lm_stamps = torch.zeros(8 * (self.LM_RECORD_CAPACITY + 2), dtype=torch.int64,
                                     device=self.device)

        def stamp(slot):
            N.check(self.lib.pba_diag_lm_stamp(self._lm_state.data_ptr(), self.lm_stamps.data_ptr(),
                                               slot, stream.cuda_stream), "pba_diag_lm_stamp")
        return stamp

    def __del__(self):
        loop = getattr(self, "_lm_loop", None)
        if loop is not None and getattr(loop, "value", None):
            try:
                self.lib.pba_lm_loop_destroy(loop)
            except Exception:
                pass

    def accept(self) -> None:
        self.cur = 1 - self.cur

    def current_rows(self):
        return (self.poses[self.cur].cpu().numpy().copy(),
                self.gens[self.cur].cpu().numpy().copy())

    def cost_only(self, rows: np.ndarray):
        """total_error path: cost/count without Jacobians (solver.py:655-670)."""
        poses = torch.from_numpy(np.ascontiguousarray(rows, dtype=np.float64)).to(self.device)
        recs = self.linearize(poses, want_jacobians=False)
        self.sum_totals(recs, self._scal[0:2])
        vals, _ = self._read_scalars()
        return float(vals[0]), int(round(vals[1]))
