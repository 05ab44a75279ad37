"""Five-channel cue images and pyramids of the drop-in API.

Mirrors `CueImage`, `CuePyramid` and the pyramid index map of the reference
(pkg/src/photoba/cues.py:84-166, 254-261).  A cue image stacks intensity,
depth/range and a unit-normal field; the derived validity masks and
central-difference gradients follow cues.py:106-147 exactly (they are also
rebuilt on the device by csrc/texels.cu when a frame is uploaded, and the
two are checked against each other and against the reference).

`DeviceCueImage` is the GPU-resident variant used when frames are produced
on the device (synthetic benchmarks): it holds torch CUDA tensors and only
materialises host arrays on request.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .camera import Intrinsics, unproject

NORMAL_COHERENCE_MIN_DOT = 0.9  # cues.py:44


class PyramidConfigError(ValueError):
    """Bad scale list for pyramid construction (cues.py:22-23)."""


def _interior(a: np.ndarray) -> np.ndarray:
    return a[1:-1, 1:-1]


def _four_neighbours(a: np.ndarray):
    """(right, left, down, up) neighbours of every interior pixel."""
    return a[1:-1, 2:], a[1:-1, :-2], a[2:, 1:-1], a[:-2, 1:-1]


def central_gradients(values: np.ndarray, valid: np.ndarray):
    """[d/dcol, d/drow] half central differences, zero unless the pixel and its
    4-neighbourhood are valid; the border never has a gradient (cues.py:63-81)."""
    ok = np.zeros(valid.shape, dtype=bool)
    inner = _interior(valid).copy()
    for nb in _four_neighbours(valid):
        inner &= nb
    ok[1:-1, 1:-1] = inner
    grad = np.zeros(values.shape + (2,))
    right, left, down, up = _four_neighbours(values)
    grad[1:-1, 1:-1, ..., 0] = 0.5 * (right - left)
    grad[1:-1, 1:-1, ..., 1] = 0.5 * (down - up)
    grad[~ok] = 0.0
    return grad, ok


def neighbour_coherence(normals: np.ndarray, valid: np.ndarray) -> np.ndarray:
    """Interior pixels whose four neighbours' normals agree (dot >= 0.9)."""
    ok = np.zeros(valid.shape, dtype=bool)
    c = _interior(normals)
    agree = np.ones(c.shape[:2], dtype=bool)
    for nb in _four_neighbours(normals):
        dot = (c[..., 0] * nb[..., 0] + c[..., 1] * nb[..., 1]) + c[..., 2] * nb[..., 2]
        agree &= dot >= NORMAL_COHERENCE_MIN_DOT
    ok[1:-1, 1:-1] = agree
    return ok


_DERIVED = ("depth_valid", "normal_valid", "grad_intensity", "grad_depth", "grad_normals",
            "sampleable_intensity", "sampleable_depth", "sampleable_normals")


@dataclass
class CueImage:
    """Intensity in [0,1], depth/range in metres, normals; masks derived eagerly."""

    intensity: np.ndarray
    depth: np.ndarray
    normals: np.ndarray
    intrinsics: Intrinsics

    depth_valid: np.ndarray = field(init=False, repr=False)
    normal_valid: np.ndarray = field(init=False, repr=False)
    grad_intensity: np.ndarray = field(init=False, repr=False)
    grad_depth: np.ndarray = field(init=False, repr=False)
    grad_normals: np.ndarray = field(init=False, repr=False)
    sampleable_intensity: np.ndarray = field(init=False, repr=False)
    sampleable_depth: np.ndarray = field(init=False, repr=False)
    sampleable_normals: np.ndarray = field(init=False, repr=False)

    def __post_init__(self) -> None:
        inten = np.asarray(self.intensity, dtype=float)
        h, w = inten.shape
        depth = np.array(self.depth, dtype=float)
        normals = np.array(self.normals, dtype=float)
        if depth.shape != (h, w) or normals.shape != (h, w, 3):
            raise ValueError("cue channel shapes disagree")
        cam = self.intrinsics
        if (cam.height, cam.width) != (h, w):
            raise ValueError("intrinsics do not match image size")
        with np.errstate(invalid="ignore"):
            out_of_range = ~np.isfinite(depth) | (depth < cam.depth_min) | (depth > cam.depth_max)
        depth[out_of_range] = 0.0
        depth_valid = depth > 0.0
        nrm = np.sqrt((normals[..., 0] ** 2 + normals[..., 1] ** 2) + normals[..., 2] ** 2)
        normal_valid = (nrm > 0.5) & depth_valid
        normals[~normal_valid] = 0.0
        g_i, ok_i = central_gradients(inten, depth_valid)
        g_d, ok_d = central_gradients(depth, depth_valid)
        coherent = normal_valid & neighbour_coherence(normals, normal_valid)
        g_n, ok_n = central_gradients(normals, coherent)
        fields = dict(intensity=inten, depth=depth, normals=normals, depth_valid=depth_valid,
                      normal_valid=normal_valid, grad_intensity=g_i, grad_depth=g_d,
                      grad_normals=g_n, sampleable_intensity=ok_i, sampleable_depth=ok_d,
                      sampleable_normals=ok_n)
        for name, arr in fields.items():
            arr = np.array(arr, copy=True) if not arr.flags.owndata else arr
            arr.flags.writeable = False
            setattr(self, name, arr)

    @property
    def shape(self) -> tuple[int, int]:
        return self.intensity.shape


class DeviceCueImage:
    """A cue image whose channels live on the GPU as torch tensors.

    Used for device-generated inputs (the synthetic benchmark path); the
    device store consumes the tensors directly.  Host arrays are produced
    lazily, e.g. `depth_valid` for graph construction.
    """

    def __init__(self, intensity, depth, normals, intrinsics: Intrinsics):
        self.device_intensity = intensity
        self.device_depth = depth
        self.device_normals = normals
        self.intrinsics = intrinsics
        self._host: CueImage | None = None
        self._depth: np.ndarray | None = None

    @property
    def shape(self) -> tuple[int, int]:
        return tuple(self.device_intensity.shape)

    def host(self) -> CueImage:
        if self._host is None:
            self._host = CueImage(self.device_intensity.cpu().numpy(),
                                  self.device_depth.cpu().numpy(),
                                  self.device_normals.cpu().numpy(), self.intrinsics)
        return self._host

    @property
    def depth_valid(self) -> np.ndarray:
        d = self.device_depth
        cam = self.intrinsics
        ok = (d >= cam.depth_min) & (d <= cam.depth_max) & (d > 0)
        return ok.cpu().numpy()

    @property
    def depth(self) -> np.ndarray:
        """The clamped depth of CueImage.__post_init__ (out-of-range or
        non-finite -> 0) without building the whole host image (graph
        construction only needs depth and depth_valid)."""
        if self._host is not None:
            return self._host.depth
        if self._depth is None:
            d = np.array(self.device_depth.cpu().numpy(), dtype=float)
            cam = self.intrinsics
            with np.errstate(invalid="ignore"):
                bad = ~np.isfinite(d) | (d < cam.depth_min) | (d > cam.depth_max)
            d[bad] = 0.0
            d.flags.writeable = False
            self._depth = d
        return self._depth

    def __getattr__(self, name):
        if name in _DERIVED or name in ("intensity", "normals"):
            return getattr(self.host(), name)
        raise AttributeError(name)


@dataclass(frozen=True)
class CuePyramid:
    """Cue images of one view, coarsest level first."""

    levels: tuple
    scales: tuple

    def __post_init__(self) -> None:
        if len(self.levels) != len(self.scales):
            raise ValueError("levels and scales disagree")

    def __len__(self) -> int:
        return len(self.levels)


def footprint_index(h: int, w: int, s: float):
    """Flat output index of every source pixel under u_out = floor(u * s),
    the kept mask and the output size (cues.py:254-261; bit-exact)."""
    out_h, out_w = int(math.floor(h * s)), int(math.floor(w * s))
    rows = np.floor(np.arange(h) * s).astype(np.int64)
    cols = np.floor(np.arange(w) * s).astype(np.int64)
    keep = (rows[:, None] < out_h) & (cols[None, :] < out_w)
    return rows[:, None] * out_w + cols[None, :], keep, out_h, out_w


def validate_scales(scales) -> tuple:
    scales = tuple(float(s) for s in scales)
    if not scales:
        raise PyramidConfigError("need at least one pyramid scale")
    if any(not 0.0 < s <= 1.0 for s in scales):
        raise PyramidConfigError(f"scales must lie in (0, 1], got {scales}")
    if any(b <= a for a, b in zip(scales, scales[1:])):
        raise PyramidConfigError(f"scales must increase toward the finest level, got {scales}")
    return scales


def downscale_cues(intensity, depth, normals, depth_ok, normal_ok, s):
    """One pyramid level (cues.py:278-326): valid-mean intensity (plain mean
    when a footprint has no valid return), lower-median depth, averaged and
    renormalised normals (dropped when incoherent)."""
    h, w = depth.shape
    idx, keep, out_h, out_w = footprint_index(h, w, s)
    n_out = out_h * out_w
    flat = idx[keep]
    dok = depth_ok[keep]
    nok = normal_ok[keep]
    vals = np.asarray(intensity, dtype=float)[keep]
    sum_v = np.bincount(flat[dok], weights=vals[dok], minlength=n_out)
    cnt_v = np.bincount(flat[dok], minlength=n_out)
    sum_a = np.bincount(flat, weights=vals, minlength=n_out)
    cnt_a = np.bincount(flat, minlength=n_out)
    out_i = np.where(cnt_v > 0, sum_v / np.maximum(cnt_v, 1), sum_a / np.maximum(cnt_a, 1))
    # lower median of each footprint's valid depths
    grp = flat[dok]
    dv = np.asarray(depth, dtype=float)[keep][dok]
    order = np.lexsort((dv, grp))
    g_sorted, d_sorted = grp[order], dv[order]
    lo = np.searchsorted(g_sorted, np.arange(n_out), side="left")
    hi = np.searchsorted(g_sorted, np.arange(n_out), side="right")
    out_d = np.zeros(n_out)
    has = hi > lo
    out_d[has] = d_sorted[lo[has] + (hi[has] - lo[has] - 1) // 2]
    # normals: mean of valid normals, renormalised where coherent
    cnt_n = np.bincount(flat[nok], minlength=n_out)
    mean_n = np.zeros((n_out, 3))
    for k in range(3):
        mean_n[:, k] = np.bincount(flat[nok], weights=np.asarray(normals)[..., k][keep][nok],
                                   minlength=n_out)
    with np.errstate(invalid="ignore", divide="ignore"):
        mean_n = mean_n / np.maximum(cnt_n, 1)[:, None]
    nrm = np.linalg.norm(mean_n, axis=-1)
    good = (cnt_n > 0) & (nrm >= 0.5)
    unit = np.zeros_like(mean_n)
    unit[good] = mean_n[good] / nrm[good, None]
    return out_i.reshape(out_h, out_w), out_d.reshape(out_h, out_w), unit.reshape(out_h, out_w, 3)


SAMPLE_CHANNELS = ("intensity", "depth", "normals")


def _footprint(img, uv: np.ndarray):
    """Bilinear footprint of continuous pixels (cues.py:397-405): inside iff
    0 <= x <= W-1 and 0 <= y <= H-1; top-left corner clipped to W-2 / H-2 so
    the last row / column interpolate with weight 1; outside points read
    corner (0, 0) with zero weights."""
    h, w = img.shape
    x, y = uv[..., 0], uv[..., 1]
    inside = (x >= 0.0) & (x <= w - 1.0) & (y >= 0.0) & (y <= h - 1.0)
    cx = np.clip(np.floor(np.where(inside, x, 0.0)).astype(int), 0, w - 2)
    cy = np.clip(np.floor(np.where(inside, y, 0.0)).astype(int), 0, h - 2)
    fx = np.where(inside, x - cx, 0.0)
    fy = np.where(inside, y - cy, 0.0)
    return inside, cx, cy, fx, fy


def _interp(arr: np.ndarray, cx, cy, fx, fy) -> np.ndarray:
    """(1-fy)((1-fx) a00 + fx a01) + fy((1-fx) a10 + fx a11), broadcast over
    trailing channel axes (cues.py:385-394, same association)."""
    a00, a01 = arr[cy, cx], arr[cy, cx + 1]
    a10, a11 = arr[cy + 1, cx], arr[cy + 1, cx + 1]
    tail = (1,) * (a00.ndim - np.ndim(fx))
    fx = np.reshape(fx, np.shape(fx) + tail)
    fy = np.reshape(fy, np.shape(fy) + tail)
    return (1.0 - fy) * ((1.0 - fx) * a00 + fx * a01) + fy * ((1.0 - fx) * a10 + fx * a11)


def sample(img, uv, channel: str):
    """Bilinear value and gradient of one cue channel at continuous pixels
    (the reference's public `sample`, cues.py:412-430): (value, gradient,
    valid).  The gradient interpolates the precomputed central-difference
    image; a lookup is valid only when it is inside and all four corners
    are sampleable for that channel.  A single (2,) pixel returns scalars
    (a bool validity).  Host numpy, like the reference: this is a per-call
    utility, not part of the per-iteration path (which samples in K1)."""
    if channel not in SAMPLE_CHANNELS:
        raise ValueError(f"unknown channel {channel!r}")
    pts = np.asarray(uv, dtype=float)
    one = pts.ndim == 1
    pts = np.atleast_2d(pts)
    inside, cx, cy, fx, fy = _footprint(img, pts)
    ok_map = getattr(img, "sampleable_" + channel)
    ok = inside & ok_map[cy, cx] & ok_map[cy, cx + 1] & ok_map[cy + 1, cx] & ok_map[cy + 1, cx + 1]
    val = _interp(getattr(img, channel), cx, cy, fx, fy)
    grad = _interp(getattr(img, "grad_" + channel), cx, cy, fx, fy)
    if one:
        return val[0], grad[0], bool(ok[0])
    return val, grad, ok


@dataclass(frozen=True)
class NormalConfig:
    """Plane-fit normal estimation parameters (cues.py:26-39): Chebyshev
    window half-width round(k_tau / depth) clamped to [radius_min,
    radius_max], at least `min_points` valid neighbours, and a middle
    eigenvalue above degeneracy_ratio x the largest."""

    k_tau: float = 4.0
    radius_min: float = 2.0
    radius_max: float = 8.0
    min_points: int = 6
    degeneracy_ratio: float = 1e-4


def _moment_integral(points: np.ndarray, valid: np.ndarray) -> np.ndarray:
    """(h+1, w+1, 10) summed-area table of [x y z xx xy xz yy yz zz 1] over
    valid pixels.  Column-wise then row-wise running sums, the summation
    order of cues.py:174-176, so window sums round identically."""
    h, w = valid.shape
    m = np.zeros((h, w, 10))
    x, y, z = (np.where(valid, points[..., k], 0.0) for k in range(3))
    m[..., 0], m[..., 1], m[..., 2] = x, y, z
    px, py, pz = points[..., 0], points[..., 1], points[..., 2]
    for k, (a, b) in enumerate(((px, px), (px, py), (px, pz), (py, py), (py, pz), (pz, pz))):
        m[..., 3 + k] = np.where(valid, a * b, 0.0)
    m[..., 9] = valid
    sat = np.zeros((h + 1, w + 1, 10))
    sat[1:, 1:] = np.cumsum(np.cumsum(m, axis=0), axis=1)
    return sat


def estimate_normals(depth: np.ndarray, cam: Intrinsics, cfg: NormalConfig | None = None) -> np.ndarray:
    """Observer-facing unit normals from a depth/range image (cues.py:187-246).

    Each valid pixel fits a least-squares plane to the points of its
    depth-adaptive window (smallest eigenvector of the window's scatter
    matrix); too few neighbours, a degenerate (line-like) fit, a grazing fit
    or a non-finite result leave the zero vector.  All pixels are handled in
    one batch: per-pixel half-widths index the shared summed-area table.
    """
    cfg = cfg or NormalConfig()
    depth = np.asarray(depth, dtype=float)
    out = np.zeros(depth.shape + (3,))
    rr, cc, S, p = window_scatter(depth, cam, cfg)
    if rr.size == 0:
        return out
    n, ok = plane_normals(S, p, cfg.degeneracy_ratio)
    out[rr[ok], cc[ok]] = n[ok]
    return out


def window_scatter(depth: np.ndarray, cam: Intrinsics, cfg: NormalConfig):
    """Pixels with enough valid window neighbours (rows, cols), their window
    scatter matrices S (k, 3, 3) and points p (k, 3) — estimate_normals up
    to the eigen step (cues.py:187-238)."""
    depth = np.asarray(depth, dtype=float)
    h, w = depth.shape
    empty = (np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros((0, 3, 3)), np.zeros((0, 3)))
    with np.errstate(invalid="ignore"):
        valid = np.isfinite(depth) & (depth >= cam.depth_min) & (depth <= cam.depth_max)
    if not valid.any():
        return empty
    pts = np.zeros((h, w, 3))
    rr, cc = np.nonzero(valid)
    pts[rr, cc] = unproject(cam, np.stack([cc.astype(float), rr.astype(float)], axis=-1),
                            depth[rr, cc])
    sat = _moment_integral(pts, valid)
    half = np.clip(np.round(cfg.k_tau / depth[rr, cc]), cfg.radius_min, cfg.radius_max).astype(np.int64)
    top, bot = np.clip(rr - half, 0, h), np.clip(rr + half + 1, 0, h)
    lft, rgt = np.clip(cc - half, 0, w), np.clip(cc + half + 1, 0, w)
    win = sat[bot, rgt] - sat[top, rgt] - sat[bot, lft] + sat[top, lft]
    cnt = win[:, 9]
    use = cnt >= cfg.min_points
    rr, cc, win, cnt = rr[use], cc[use], win[use], cnt[use]
    if rr.size == 0:
        return empty
    mu = win[:, 0:3] / cnt[:, None]
    # scatter[i][j] = S_ij - (count * mu_i) * mu_j, entry by entry (the
    # lower triangle is what the symmetric eigensolver reads)
    S = win[:, (3, 4, 5, 4, 6, 7, 5, 7, 8)].reshape(-1, 3, 3)
    S = S - (cnt[:, None] * mu)[:, :, None] * mu[:, None, :]
    return rr, cc, S, pts[rr, cc]


def plane_normals(S: np.ndarray, p: np.ndarray, degeneracy_ratio: float):
    """The eigen step and gates of estimate_normals (cues.py:239-245) for a
    stack of scatter matrices S (k, 3, 3; eigh reads the lower triangle) and
    their points p (k, 3): the observer-facing smallest eigenvector and
    whether it passes the planarity, grazing and finiteness gates.  The GPU
    builder (pyramid_device.py) calls this for the pixels it cannot decide."""
    lam, vec = np.linalg.eigh(S)
    n = vec[:, :, 0]
    planar = lam[:, 1] > np.maximum(degeneracy_ratio * lam[:, 2], 0.0)
    facing = np.einsum("ij,ij->i", n, p)
    n = np.where(facing[:, None] > 0.0, -n, n)
    ok = planar & (np.abs(facing) > 1e-12) & np.isfinite(n).all(axis=1)
    return n, ok


def build_cue_image(intensity, depth, cam: Intrinsics, cfg: NormalConfig | None = None,
                    normals=None) -> CueImage:
    """Full-resolution cue image, estimating normals unless given (cues.py:329-339)."""
    if normals is None:
        normals = estimate_normals(depth, cam, cfg)
    return CueImage(intensity, depth, normals, cam)


def build_pyramid(intensity, depth, cam: Intrinsics, scales=(0.125, 0.25, 0.5),
                  cfg: NormalConfig | None = None, device=None) -> CuePyramid:
    """Cue pyramid of one intensity/depth pair (cues.py:342-375): normals
    estimated once at full resolution, then each level downscaled per
    channel; `scales` coarsest to finest in (0, 1].  With `device` (e.g.
    "cuda") the pyramid is built by the GPU kernels of pyramid_device.py and
    its levels are DeviceCueImage."""
    if device is not None:
        from .pyramid_device import build_pyramids_device
        return build_pyramids_device(intensity, depth, cam, scales, cfg, device)[0]
    scales = validate_scales(scales)
    if np.shape(intensity) != np.shape(depth):
        raise ValueError("intensity and depth shapes disagree")
    depth = np.where(np.isfinite(depth), depth, 0.0)
    return build_pyramid_from_normals(intensity, depth, estimate_normals(depth, cam, cfg), cam,
                                      scales)


def build_pyramid_from_normals(intensity, depth, normals, cam: Intrinsics, scales) -> CuePyramid:
    """Pyramid from full-resolution cues with given normals (cues.py:342-375,
    with the normal-estimation step replaced by the provided field)."""
    scales = validate_scales(scales)
    depth = np.where(np.isfinite(depth), depth, 0.0)
    depth_ok = (depth >= cam.depth_min) & (depth <= cam.depth_max)
    normal_ok = np.linalg.norm(normals, axis=-1) > 0.5
    levels = []
    for s in scales:
        li, ld, ln = downscale_cues(intensity, depth, normals, depth_ok, normal_ok, s)
        levels.append(CueImage(li, ld, ln, cam.scaled(s)))
    return CuePyramid(tuple(levels), scales)
