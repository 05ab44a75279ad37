"""Synthetic box-scene frames for tests and benchmarks (torch, CPU or GPU).

The reference ships a numpy ray caster (pkg/src/photoba/synthetic.py) that
is far too slow for the 1000-scan benchmark configuration (~12 min,
SURVEY.md App. C).  This module renders the same kind of scene — the
inside of an axis-aligned box with band-limited sine albedo, Lambert
shading plus ambient — as batched tensor ops, so a 1000 x 128 x 1024 LiDAR
sequence is generated on the GPU in seconds.  Normals are the analytic
surface normals (the reference estimates them from depth by plane fits,
cues.py:187-246); pyramids use the reference's downscale rules
(cues.py:278-326) for the integer 2x / 4x footprints of the benchmark
scales.  This is input generation only — nothing here is on the hot path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .camera import PINHOLE, SPHERICAL, Intrinsics
from .cueimage import CueImage, CuePyramid, DeviceCueImage, build_pyramid_from_normals
from .se3 import PerturbationVector, Pose, exp


@dataclass(frozen=True)
class BoxScene:
    low: tuple = (-3.0, -3.0, -3.0)
    high: tuple = (3.0, 3.0, 3.0)
    albedo: float = 0.85
    frequency: tuple = (2.1, 1.7, 2.9)
    phase: tuple = (0.4, 1.3, 2.2)
    amplitude: float = 0.45
    light: tuple = (0.3, -0.5, -0.8)
    ambient: float = 0.35


def corridor_scene(length: float) -> BoxScene:
    """The App. C corridor: box (-10,-4,-2.5) .. (length, 4, 4)."""
    return BoxScene(low=(-10.0, -4.0, -2.5), high=(float(length), 4.0, 4.0))


def unit_rays(cam: Intrinsics, device, dtype=torch.float64) -> torch.Tensor:
    """(H*W, 3) ray directions scaled so the hit parameter is z-depth (pinhole)
    or range (spherical), i.e. unproject(cam, uv, 1)."""
    u = torch.arange(cam.width, device=device, dtype=dtype)
    v = torch.arange(cam.height, device=device, dtype=dtype)
    a = (u - cam.cx) / cam.fx
    e = (v - cam.cy) / cam.fy
    A = a[None, :].expand(cam.height, cam.width)
    E = e[:, None].expand(cam.height, cam.width)
    if cam.model == PINHOLE:
        d = torch.stack([A, E, torch.ones_like(A)], dim=-1)
    else:
        ce = torch.cos(E)
        d = torch.stack([ce * torch.cos(A), ce * torch.sin(A), torch.sin(E)], dim=-1)
    return d.reshape(-1, 3)


def render_batch(scene: BoxScene, cam: Intrinsics, sensor_poses: torch.Tensor, rays=None):
    """Render B views from inside the box.  sensor_poses: (B, 12) rows.
    Returns intensity (B,H,W), depth (B,H,W), normals (B,H,W,3) (sensor frame)."""
    dev, dt = sensor_poses.device, sensor_poses.dtype
    if rays is None:
        rays = unit_rays(cam, dev, dt)
    B = sensor_poses.shape[0]
    R = sensor_poses[:, :9].reshape(B, 3, 3)
    o = sensor_poses[:, 9:12]
    dw = torch.einsum("bij,pj->bpi", R, rays)  # world directions
    low = torch.tensor(scene.low, device=dev, dtype=dt)
    high = torch.tensor(scene.high, device=dev, dtype=dt)
    # exit distance through the wall each axis is heading to
    wall = torch.where(dw > 0, high, low)
    with torch.no_grad():
        tax = (wall - o[:, None, :]) / dw
    tax = torch.where(dw.abs() > 1e-12, tax, torch.full_like(tax, math.inf))
    tax = torch.where(tax > 1e-9, tax, torch.full_like(tax, math.inf))
    t, axis = tax.min(dim=-1)
    hit_p = o[:, None, :] + t[..., None] * dw
    n = torch.zeros_like(dw)
    sgn = -torch.sign(torch.gather(dw, -1, axis[..., None]))
    n.scatter_(-1, axis[..., None], sgn)
    f = torch.tensor(scene.frequency, device=dev, dtype=dt)
    ph = torch.tensor(scene.phase, device=dev, dtype=dt)
    s = torch.sin(hit_p * f + ph).sum(-1) / 3.0
    albedo = torch.clamp(scene.albedo * (1.0 + scene.amplitude * s), 0.05, 1.0)
    light = torch.tensor(scene.light, device=dev, dtype=dt)
    light = light / torch.linalg.norm(light)
    lam = torch.clamp(-(n @ light), min=0.0)
    inten = torch.clamp(albedo * (scene.ambient + (1.0 - scene.ambient) * lam), 0.0, 1.0)
    ok = torch.isfinite(t) & (t >= cam.depth_min) & (t <= cam.depth_max)
    depth = torch.where(ok, t, torch.zeros_like(t))
    inten = torch.where(ok, inten, torch.zeros_like(inten))
    n_sensor = torch.einsum("bpi,bij->bpj", n, R)  # R^T n
    n_sensor = torch.where(ok[..., None], n_sensor, torch.zeros_like(n_sensor))
    H, W = cam.height, cam.width
    return inten.reshape(B, H, W), depth.reshape(B, H, W), n_sensor.reshape(B, H, W, 3)


def downscale_block(inten, depth, normals, cam: Intrinsics, k: int):
    """Integer-factor (k x k footprint) version of the reference downscale
    rules on tensors (B,H,W): valid-mean intensity, lower median of valid
    depths, renormalised mean normal (cues.py:278-326)."""
    B, H, W = depth.shape
    h, w = H // k, W // k
    d = depth[:, : h * k, : w * k].reshape(B, h, k, w, k).permute(0, 1, 3, 2, 4).reshape(B, h, w, k * k)
    i = inten[:, : h * k, : w * k].reshape(B, h, k, w, k).permute(0, 1, 3, 2, 4).reshape(B, h, w, k * k)
    nn = normals[:, : h * k, : w * k].reshape(B, h, k, w, k, 3).permute(0, 1, 3, 2, 4, 5)
    nn = nn.reshape(B, h, w, k * k, 3)
    dok = (d >= cam.depth_min) & (d <= cam.depth_max)
    cnt = dok.sum(-1)
    isum = torch.where(dok, i, torch.zeros_like(i)).sum(-1)
    out_i = torch.where(cnt > 0, isum / cnt.clamp(min=1), i.mean(-1))
    ds = torch.where(dok, d, torch.full_like(d, math.inf)).sort(-1).values
    idx = ((cnt - 1).clamp(min=0) // 2)[..., None]
    out_d = torch.where(cnt > 0, torch.gather(ds, -1, idx)[..., 0], torch.zeros_like(out_i))
    nok = torch.linalg.norm(nn, dim=-1) > 0.5
    ncnt = nok.sum(-1)
    nsum = torch.where(nok[..., None], nn, torch.zeros_like(nn)).sum(-2)
    mean = nsum / ncnt.clamp(min=1)[..., None]
    nrm = torch.linalg.norm(mean, dim=-1)
    good = (ncnt > 0) & (nrm >= 0.5)
    unit = torch.where(good[..., None], mean / nrm.clamp(min=1e-300)[..., None],
                       torch.zeros_like(mean))
    return out_i, out_d, unit


def corridor_trajectory(n: int, spacing: float) -> list:
    """App. C poses: t = (s k, 0.6 sin 0.21k, 0.1 cos 0.13k), yaw 0.15 sin 0.37k."""
    poses = []
    for k in range(n):
        yaw = 0.15 * math.sin(0.37 * k)
        r = exp(PerturbationVector([0, 0, 0], [0, 0, math.sin(yaw / 2)])).rotation
        poses.append(Pose(r, [spacing * k, 0.6 * math.sin(0.21 * k), 0.1 * math.cos(0.13 * k)]))
    return poses


def room_loop(n: int) -> list:
    """Poses wandering inside the 6 m room (pkg/tests/rigs.py:39-52 recipe)."""
    poses = []
    for k in range(n):
        a = 2.0 * math.pi * k / n
        yaw = 0.25 * math.sin(2 * a)
        pitch = 0.1 * math.cos(a)
        r = (exp(PerturbationVector([0, 0, 0], [0, math.sin(pitch / 2), 0])).rotation
             @ exp(PerturbationVector([0, 0, 0], [0, 0, math.sin(yaw / 2)])).rotation)
        poses.append(Pose(r, [0.8 * math.cos(a), 0.5 * math.sin(a), -0.4 + 0.05 * k]))
    return poses


def perturb(poses, sigma_t: float, sigma_r: float, seed: int, keep_first: bool = True) -> list:
    """Seeded Gaussian SE(3) noise (the perturb_trajectory recipe, synthetic.py:240-254)."""
    rng = np.random.default_rng(seed)
    out = []
    for k, p in enumerate(poses):
        if keep_first and k == 0:
            out.append(p)
            continue
        dt = rng.normal(0.0, sigma_t, 3)
        dq = rng.normal(0.0, sigma_r / 2.0, 3)
        out.append(p.compose(exp(PerturbationVector(dt, dq))))
    return out


def sensor_rows(platform_poses, ext: Pose) -> torch.Tensor:
    rows = np.stack([p.compose(ext).as_row() for p in platform_poses])
    return torch.from_numpy(rows)


def host_pyramids(scene, cam, platform_poses, ext: Pose, scales) -> list:
    """Reference-style host pyramids (numpy CueImages) for small problems."""
    rows = sensor_rows(platform_poses, ext)
    inten, depth, normals = render_batch(scene, cam, rows)
    out = []
    for b in range(rows.shape[0]):
        out.append(build_pyramid_from_normals(inten[b].numpy(), depth[b].numpy(),
                                              normals[b].numpy(), cam, scales))
    return out


def device_pyramids(scene, cam, platform_poses, ext: Pose, factors, device, batch: int = 64,
                    normals: str = "estimate"):
    """GPU pyramids (DeviceCueImage levels) for large problems.  `factors`
    are integer downscale factors coarsest first, e.g. (4, 2, 1).  With
    normals="estimate" (default) the rendered intensity/depth go through the
    device pyramid builder (pyramid_device.py: plane-fit normals + the
    reference downscale, as build_pyramid does, cues.py:342-375); "analytic"
    uses the renderer's exact surface normals instead."""
    rows = sensor_rows(platform_poses, ext).to(device)
    rays = unit_rays(cam, device)
    scales = tuple(1.0 / f for f in factors)
    pyrs = []
    for s0 in range(0, rows.shape[0], batch):
        inten, depth, nrm_true = render_batch(scene, cam, rows[s0:s0 + batch], rays)
        if normals == "estimate":
            from .pyramid_device import build_pyramids_device
            pyrs.extend(build_pyramids_device(inten, depth, cam, scales, device=device))
            continue
        per_level = []
        for f in factors:
            lc = cam.scaled(1.0 / f)
            if f == 1:
                li, ld = inten, depth
                nrm = torch.linalg.norm(nrm_true, dim=-1, keepdim=True)
                ln = torch.where(nrm > 0.5, nrm_true / nrm.clamp(min=1e-300),
                                 torch.zeros_like(nrm_true))
            else:
                li, ld, ln = downscale_block(inten, depth, nrm_true, cam, f)
            per_level.append((lc, li, ld, ln))
        for b in range(inten.shape[0]):
            levels = tuple(DeviceCueImage(li[b].contiguous(), ld[b].contiguous(),
                                          ln[b].contiguous(), lc) for (lc, li, ld, ln) in per_level)
            pyrs.append(CuePyramid(levels, scales))
    return pyrs


def lidar_os0_128(width: int = 1024, height: int = 128) -> Intrinsics:
    """OS0-128-shaped spherical sensor (pkg/tests/rigs.py:23-26 lidar_cam)."""
    return Intrinsics(width / (2.0 * math.pi), height / (math.pi / 2.0), width / 2.0, height / 2.0,
                      width, height, SPHERICAL, 0.2, 80.0)


def hdl64(width: int = 1024, height: int = 64) -> Intrinsics:
    """HDL-64-shaped spherical sensor of App. C config 2."""
    fy = height / math.radians(26.9)
    return Intrinsics(width / (2 * math.pi), fy, width / 2.0, fy * math.radians(24.9), width,
                      height, SPHERICAL, 0.5, 80.0)


def tum_640() -> Intrinsics:
    """TUM-shaped 640x480 RGB-D camera of App. C configs 3 and 5."""
    return Intrinsics(525.0, 525.0, 319.5, 239.5, 640, 480, PINHOLE, 0.1, 20.0)


def rgbd_160() -> Intrinsics:
    """App. C config 1 pinhole camera."""
    return Intrinsics(70.0, 70.0, 80.0, 60.0, 160, 120, PINHOLE, 0.1, 50.0)
