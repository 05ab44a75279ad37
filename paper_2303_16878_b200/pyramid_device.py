"""Cue-pyramid construction on the GPU (K6, csrc/pyramid.cu).

Device counterpart of `build_pyramid` / `estimate_normals` (reference
pkg/src/photoba/cues.py:187-246, 278-326, 342-375; host restatement in
cueimage.py).  Frames of one camera are processed in batches: the moment
summed-area table, the per-pixel plane fits and every downscaled level stay
in HBM and come out as `DeviceCueImage` levels, which the device frame store
turns into texels without a host round trip.

Parity: intensity, depth and the downscale are bit-equal to the reference;
normals agree to the eigen-solver's precision (Jacobi vs LAPACK), see
pyramid.cu and DESIGN.md.
"""

from __future__ import annotations

import torch

from . import native as N
from .camera import Intrinsics, ray_table
from .cueimage import CuePyramid, DeviceCueImage, NormalConfig, footprint_index, validate_scales
from .device import camera_struct

_SCRATCH_BUDGET = 1 << 30  # bytes of moment table per batch


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _as_batch(x, device) -> torch.Tensor:
    t = torch.as_tensor(x, dtype=torch.float64)
    if t.dim() == 2:
        t = t[None]
    if t.dim() != 3:
        raise ValueError("expected (H, W) or (n, H, W) images")
    return t.to(device).contiguous()


def _config(cfg: NormalConfig | None) -> N.NormalConfigC:
    cfg = cfg or NormalConfig()
    return N.NormalConfigC(float(cfg.k_tau), float(cfg.radius_min), float(cfg.radius_max),
                           float(cfg.min_points), float(cfg.degeneracy_ratio))


def _frames_per_batch(lib, cs, n: int) -> int:
    per = int(lib.pba_normals_scratch_bytes(cs, 1))
    return max(1, min(n, 65535, _SCRATCH_BUDGET // max(per, 1)))


def estimate_normals_device(depth, cam: Intrinsics, cfg: NormalConfig | None = None,
                            device=None) -> torch.Tensor:
    """estimate_normals (cues.py:187-246) of (H, W) or (n, H, W) depth/range
    images on the GPU; returns (.., H, W, 3) fp64 normals on the device."""
    lib = N.load()
    device = torch.device(device or (depth.device if torch.is_tensor(depth) and depth.is_cuda
                                     else "cuda"))
    squeeze = torch.as_tensor(depth).dim() == 2
    d = _as_batch(depth, device)
    n, H, W = d.shape
    if (H, W) != (cam.height, cam.width):
        raise ValueError("depth shape disagrees with the intrinsics")
    cs = camera_struct(cam)
    tab = torch.as_tensor(ray_table(cam), dtype=torch.float64, device=device)
    out = torch.empty((n, H, W, 3), dtype=torch.float64, device=device)
    cfg_c = _config(cfg)
    step = _frames_per_batch(lib, cs, n)
    scratch = torch.empty(int(lib.pba_normals_scratch_bytes(cs, min(step, n))) or 8,
                          dtype=torch.uint8, device=device)
    for f0 in range(0, n, step):
        k = min(step, n - f0)
        N.check(lib.pba_estimate_normals(cs, tab.data_ptr(), d[f0].data_ptr(), k, cfg_c,
                                         out[f0].data_ptr(), scratch.data_ptr(), _stream(device)),
                "pba_estimate_normals")
    return out[0] if squeeze else out


def downscale_cues_device(intensity: torch.Tensor, depth: torch.Tensor, normals: torch.Tensor,
                          cam: Intrinsics, s: float):
    """_downscale_cues (cues.py:278-326) of a (n, H, W) batch to scale s."""
    lib = N.load()
    n, H, W = depth.shape
    _, _, out_h, out_w = footprint_index(H, W, s)
    dev = depth.device
    oi = torch.empty((n, out_h, out_w), dtype=torch.float64, device=dev)
    od = torch.empty_like(oi)
    on = torch.empty((n, out_h, out_w, 3), dtype=torch.float64, device=dev)
    N.check(lib.pba_downscale_cues(camera_struct(cam), float(s), n, intensity.data_ptr(),
                                   depth.data_ptr(), normals.data_ptr(), out_h, out_w,
                                   oi.data_ptr(), od.data_ptr(), on.data_ptr(), _stream(dev)),
            "pba_downscale_cues")
    return oi, od, on


def build_pyramids_device(intensity, depth, cam: Intrinsics, scales=(0.125, 0.25, 0.5),
                          cfg: NormalConfig | None = None, device=None) -> list:
    """build_pyramid (cues.py:342-375) for a batch of frames of one camera:
    (n, H, W) intensity and depth (host arrays or tensors) -> n CuePyramids
    of DeviceCueImage levels resident on the GPU."""
    scales = validate_scales(scales)
    device = torch.device(device or "cuda")
    I = _as_batch(intensity, device)
    D = _as_batch(depth, device)
    if I.shape != D.shape:
        raise ValueError("intensity and depth shapes disagree")
    D = torch.where(torch.isfinite(D), D, torch.zeros((), dtype=D.dtype, device=device))
    Nrm = estimate_normals_device(D, cam, cfg, device)
    levels = []
    for s in scales:
        li, ld, ln = downscale_cues_device(I, D, Nrm, cam, s)
        levels.append((cam.scaled(s), li, ld, ln))
    return [CuePyramid(tuple(DeviceCueImage(li[b], ld[b], ln[b], lc)
                             for (lc, li, ld, ln) in levels), scales)
            for b in range(D.shape[0])]
