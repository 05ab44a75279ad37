"""Cue-pyramid construction on the GPU (K6, csrc/pyramid.cu).

Device counterpart of `build_pyramid` / `estimate_normals` (reference
pkg/src/photoba/cues.py:187-246, 278-326, 342-375; host restatement in
cueimage.py).  Frames of one camera are processed in batches: the moment
summed-area table, the per-pixel plane fits and every downscaled level stay
in HBM and come out as `DeviceCueImage` levels, which the device frame store
turns into texels without a host round trip.

Parity: intensity, depth and the downscale are bit-equal to the reference;
normal validity is bit-exact (knife-edge pixels re-decided with eigh on the
host) and the normals agree to <= 1e-10 (Jacobi vs LAPACK), see pyramid.cu
and DESIGN.md.
"""

from __future__ import annotations

import numpy as np
import torch

from . import native as N
from .camera import Intrinsics, ray_table
from .cueimage import (CuePyramid, DeviceCueImage, NormalConfig, footprint_index, plane_normals,
                       validate_scales)
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


last_recheck_count = 0  # pixels re-decided on the host by the last call (diagnostics)


def estimate_normals_device(depth, cam: Intrinsics, cfg: NormalConfig | None = None,
                            device=None, recheck_capacity: int | None = None) -> torch.Tensor:
    """estimate_normals (cues.py:187-246) of (H, W) or (n, H, W) depth/range
    images on the GPU; returns (.., H, W, 3) fp64 normals on the device.

    The 3x3 eigenproblem runs as Jacobi on the device; the pixels whose
    gates or normal could differ under numpy.linalg.eigh (reported by the
    kernel with their bit-equal scatter matrix) are decided here by the
    reference's own eigh expressions (cueimage.plane_normals), so validity
    is bit-exact and every normal matches to <= 1e-10.  recheck_capacity
    sizes the first recheck buffer (it grows to fit; tests shrink it)."""
    global last_recheck_count
    lib = N.load()
    cfg = cfg or NormalConfig()
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
    count = torch.zeros(1, dtype=torch.int32, device=device)
    cap = recheck_capacity if recheck_capacity is not None else 4096 + (min(step, n) * H * W) // 256
    last_recheck_count = 0
    recheck = torch.empty((max(cap, 1), N.NORMALS_RECHECK_DOUBLES), dtype=torch.float64,
                          device=device)
    for f0 in range(0, n, step):
        k = min(step, n - f0)
        while True:
            N.check(lib.pba_estimate_normals(cs, tab.data_ptr(), d[f0].data_ptr(), k, cfg_c,
                                             out[f0].data_ptr(), scratch.data_ptr(),
                                             recheck.data_ptr(), cap, count.data_ptr(),
                                             _stream(device)), "pba_estimate_normals")
            got = int(count.item())
            if got <= cap:
                break
            cap = got
            recheck = torch.empty((cap, N.NORMALS_RECHECK_DOUBLES), dtype=torch.float64,
                                  device=device)
        if got:
            _decide_on_host(recheck[:got], out[f0:f0 + k], cfg)
        last_recheck_count += got
    return out[0] if squeeze else out


def _decide_on_host(recheck: torch.Tensor, out: torch.Tensor, cfg: NormalConfig) -> None:
    """Re-decide the listed pixels with numpy.linalg.eigh (cues.py:239-245)."""
    rec = recheck.cpu().numpy()
    idx = rec[:, 0].astype(np.int64)
    S = np.empty((rec.shape[0], 3, 3))
    S[:, 0, 0], S[:, 1, 1], S[:, 2, 2] = rec[:, 1], rec[:, 2], rec[:, 3]
    S[:, 1, 0] = S[:, 0, 1] = rec[:, 4]
    S[:, 2, 0] = S[:, 0, 2] = rec[:, 5]
    S[:, 2, 1] = S[:, 1, 2] = rec[:, 6]
    nrm, ok = plane_normals(S, np.ascontiguousarray(rec[:, 7:10]), cfg.degeneracy_ratio)
    vals = np.where(ok[:, None], nrm, 0.0)
    flat = out.view(-1, 3)
    flat[torch.from_numpy(idx).to(out.device)] = torch.from_numpy(vals).to(out.device)


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
