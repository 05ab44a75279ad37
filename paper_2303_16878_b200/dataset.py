"""Dataset directories of the drop-in API.

Mirrors the reference's on-disk formats and loaders
(pkg/src/photoba/dataset_io.py, formats in pkg/docs/formats.md):

    manifest                         JSON: sensors, trajectory file, scales
    trajectory.txt                   `timestamp tx ty tz qx qy qz qw` lines
    <sensor>/intensity/<ts>.pgm      PGM P5, 8- or 16-bit big-endian
    <sensor>/depth/<ts>.pgm          PGM P5 16-bit, meters = raw * depth_scale

The host functions reproduce the reference bit for bit (tests/test_dataset.py
checks files written by the reference and by this module against each
other).  `load_dataset(..., device="cuda")` is the B200 path: the host only
parses headers and gathers the payloads of all frames of a sensor into one
pinned buffer; one H2D copy, one decode launch per channel (K7,
csrc/rasters.cu) and the batched pyramid builder (K6) leave every frame's
pyramid resident in HBM as DeviceCueImage levels, ready for the texel store.
"""

from __future__ import annotations

import json
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .camera import Intrinsics, SensorExtrinsics
from .cueimage import NormalConfig, build_pyramid
from .evaluation import Trajectory
from .pairgraph import FrameNode
from .se3 import Pose


class DatasetError(RuntimeError):
    """Dataset loading/saving problem (dataset_io.py:32-49)."""


class ManifestError(DatasetError):
    pass


class MissingFileError(DatasetError):
    pass


class DimensionMismatchError(DatasetError):
    pass


class TrajectoryFormatError(DatasetError):
    pass


def trajectory_from_poses(timestamps, poses) -> Trajectory:
    return Trajectory(np.asarray(timestamps, dtype=float), list(poses))


# ---------------------------------------------------------------------------
# PGM rasters
# ---------------------------------------------------------------------------

_WS = b" \t\n\r\x0b\x0c"


def _pgm_header(data: bytes, path) -> tuple[int, int, int, int]:
    """(width, height, maxval, payload offset) of a P5 file: four
    whitespace-separated tokens, '#' comments between tokens, then exactly
    one whitespace byte (dataset_io.py:79-97)."""
    tokens = []
    pos, n = 0, len(data)
    while len(tokens) < 4:
        while pos < n and data[pos] in _WS:
            pos += 1
        if pos < n and data[pos] == 0x23:  # '#': comment to end of line
            while pos < n and data[pos] != 0x0A:
                pos += 1
            continue
        start = pos
        while pos < n and data[pos] not in _WS:
            pos += 1
        tokens.append(data[start:pos])
    if tokens[0] != b"P5":
        raise DatasetError(f"{path}: not a binary PGM file")
    try:
        w, h, maxval = int(tokens[1]), int(tokens[2]), int(tokens[3])
    except ValueError:
        raise DatasetError(f"{path}: malformed PGM header") from None
    return w, h, maxval, pos + 1


def _read_payload(path):
    """(width, height, bytes per sample, payload bytes) of one raster."""
    path = Path(path)
    if not path.exists():
        raise MissingFileError(f"raster file not found: {path}")
    data = path.read_bytes()
    w, h, maxval, off = _pgm_header(data, path)
    bps = 2 if maxval > 255 else 1
    payload = data[off: off + w * h * bps]
    if len(payload) != w * h * bps:
        raise DatasetError(f"{path}: truncated raster payload")
    return w, h, bps, payload


def write_raster(path, values: np.ndarray) -> None:
    """uint8 / uint16 grid -> binary PGM (16-bit big-endian) (dataset_io.py:57-71)."""
    values = np.asarray(values)
    if values.dtype == np.uint8:
        maxval, payload = 255, values.tobytes()
    elif values.dtype == np.uint16:
        maxval, payload = 65535, values.astype(">u2").tobytes()
    else:
        raise ValueError(f"raster dtype must be uint8 or uint16, got {values.dtype}")
    h, w = values.shape
    Path(path).write_bytes(b"P5\n%d %d\n%d\n" % (w, h, maxval) + payload)


def read_raster(path) -> np.ndarray:
    """Binary PGM -> uint8 / uint16 (h, w) array (dataset_io.py:74-104)."""
    w, h, bps, payload = _read_payload(path)
    if bps == 2:
        return np.frombuffer(payload, dtype=">u2").reshape(h, w).astype(np.uint16)
    return np.frombuffer(payload, dtype=np.uint8).reshape(h, w).copy()


def write_intensity(path, intensity: np.ndarray) -> None:
    """[0, 1] intensity -> 16-bit raster of round(v * 65535) (dataset_io.py:107-110)."""
    write_raster(path, np.clip(np.round(np.asarray(intensity) * 65535.0), 0, 65535).astype(np.uint16))


def read_intensity(path) -> np.ndarray:
    raw = read_raster(path)
    return raw.astype(float) / (255.0 if raw.dtype == np.uint8 else 65535.0)


def write_depth(path, meters: np.ndarray, depth_scale: float) -> None:
    """Meters -> 16-bit raster, raw 0 = invalid (dataset_io.py:119-124)."""
    meters = np.asarray(meters, dtype=float)
    raw = np.zeros(meters.shape, dtype=np.uint16)
    with np.errstate(invalid="ignore"):
        ok = np.isfinite(meters) & (meters > 0.0)
    raw[ok] = np.clip(np.round(meters[ok] / depth_scale), 1, 65535).astype(np.uint16)
    write_raster(path, raw)


def read_depth(path, depth_scale: float) -> np.ndarray:
    raw = read_raster(path)
    if raw.dtype != np.uint16:
        raise DatasetError(f"{path}: depth rasters must be 16-bit")
    return raw.astype(float) * depth_scale


# ---------------------------------------------------------------------------
# trajectories
# ---------------------------------------------------------------------------


def save_trajectory(traj: Trajectory, path) -> None:
    """`ts tx ty tz qx qy qz qw`, 6 / 9 decimals (dataset_io.py:139-149)."""
    out = ["# timestamp tx ty tz qx qy qz qw\n"]
    for ts, pose in zip(traj.timestamps, traj.poses):
        q, t = pose.quat(), pose.translation
        out.append(f"{ts:.6f} {t[0]:.9f} {t[1]:.9f} {t[2]:.9f} "
                   f"{q[0]:.9f} {q[1]:.9f} {q[2]:.9f} {q[3]:.9f}\n")
    Path(path).write_text("".join(out))


def load_trajectory(path) -> Trajectory:
    path = Path(path)
    if not path.exists():
        raise MissingFileError(f"trajectory file not found: {path}")
    stamps, poses = [], []
    for lineno, raw in enumerate(path.read_text().splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        fields = line.split()
        if len(fields) != 8:
            raise TrajectoryFormatError(
                f"{path}:{lineno}: expected 8 fields 'ts tx ty tz qx qy qz qw', got {len(fields)}")
        try:
            vals = [float(f) for f in fields]
        except ValueError as exc:
            raise TrajectoryFormatError(f"{path}:{lineno}: {exc}") from None
        stamps.append(vals[0])
        poses.append(Pose.from_quat(np.array(vals[1:4]), np.array(vals[4:8])))
    if not stamps:
        raise TrajectoryFormatError(f"{path}: no poses found")
    try:
        return Trajectory(np.array(stamps), poses)
    except ValueError as exc:
        raise TrajectoryFormatError(f"{path}: {exc}") from None


# ---------------------------------------------------------------------------
# manifest
# ---------------------------------------------------------------------------


@dataclass
class SensorConfig:
    """One sensor entry of the manifest (dataset_io.py:186-200)."""

    sensor_id: str
    intrinsics: Intrinsics
    extrinsics: SensorExtrinsics
    depth_scale: float
    intensity_dir: str
    depth_dir: str

    def __post_init__(self) -> None:
        if self.depth_scale <= 0.0:
            raise ManifestError(f"sensor {self.sensor_id}: depth_scale must be positive")


@dataclass
class DatasetManifest:
    sensors: list
    trajectory_file: str = "trajectory.txt"
    pyramid_scales: tuple = (0.125, 0.25, 0.5)
    solver_overrides: dict = field(default_factory=dict)


_INTR_KEYS = ("model", "fx", "fy", "cx", "cy", "width", "height", "depth_min", "depth_max")


def save_manifest(manifest: DatasetManifest, path) -> None:
    sensors = []
    for s in manifest.sensors:
        k = s.intrinsics
        sensors.append({
            "sensor_id": s.sensor_id,
            "intrinsics": {key: getattr(k, key) for key in _INTR_KEYS},
            "extrinsics": {"rotation": s.extrinsics.offset.rotation.tolist(),
                           "translation": s.extrinsics.offset.translation.tolist()},
            "depth_scale": s.depth_scale,
            "intensity_dir": s.intensity_dir,
            "depth_dir": s.depth_dir,
        })
    doc = {"sensors": sensors, "trajectory": manifest.trajectory_file,
           "pyramid_scales": list(manifest.pyramid_scales), "solver": manifest.solver_overrides}
    Path(path).write_text(json.dumps(doc, indent=2) + "\n")


def load_manifest(path) -> DatasetManifest:
    path = Path(path)
    if not path.exists():
        raise MissingFileError(f"manifest not found: {path}")
    try:
        doc = json.loads(path.read_text())
    except json.JSONDecodeError as exc:
        raise ManifestError(f"{path}: {exc}") from None
    try:
        sensors = []
        for s in doc["sensors"]:
            k = s["intrinsics"]
            intr = Intrinsics(fx=float(k["fx"]), fy=float(k["fy"]), cx=float(k["cx"]),
                              cy=float(k["cy"]), width=int(k["width"]), height=int(k["height"]),
                              model=str(k["model"]), depth_min=float(k["depth_min"]),
                              depth_max=float(k["depth_max"]))
            ext = SensorExtrinsics(Pose(np.array(s["extrinsics"]["rotation"], dtype=float),
                                        np.array(s["extrinsics"]["translation"], dtype=float)))
            sensors.append(SensorConfig(str(s["sensor_id"]), intr, ext, float(s["depth_scale"]),
                                        str(s["intensity_dir"]), str(s["depth_dir"])))
        return DatasetManifest(
            sensors=sensors,
            trajectory_file=str(doc.get("trajectory", "trajectory.txt")),
            pyramid_scales=tuple(float(x) for x in doc.get("pyramid_scales", (0.125, 0.25, 0.5))),
            solver_overrides=dict(doc.get("solver", {})))
    except (KeyError, TypeError, ValueError) as exc:
        raise ManifestError(f"{path}: bad manifest entry: {exc}") from None


def timestamp_name(ts: float) -> str:
    return f"{ts:.6f}"


# ---------------------------------------------------------------------------
# loading
# ---------------------------------------------------------------------------


def _frame_paths(dataset_dir: Path, sensor: SensorConfig, ts: float):
    name = timestamp_name(ts) + ".pgm"
    ipath = dataset_dir / sensor.intensity_dir / name
    dpath = dataset_dir / sensor.depth_dir / name
    if not ipath.exists():
        raise MissingFileError(f"sensor {sensor.sensor_id}: missing intensity image {ipath}")
    if not dpath.exists():
        raise MissingFileError(f"sensor {sensor.sensor_id}: missing depth image {dpath}")
    return ipath, dpath


def _dimension_error(sensor, ts, shape):
    k = sensor.intrinsics
    return DimensionMismatchError(
        f"sensor {sensor.sensor_id} frame {timestamp_name(ts)}: image size {shape} does not "
        f"match intrinsics ({k.height}, {k.width})")


def _load_sensor_host(dataset_dir, sensor, trajectory, scales, normal_cfg):
    nodes = []
    k_int = sensor.intrinsics
    for k, (ts, pose) in enumerate(zip(trajectory.timestamps, trajectory.poses)):
        ipath, dpath = _frame_paths(dataset_dir, sensor, ts)
        inten = read_intensity(ipath)
        depth = read_depth(dpath, sensor.depth_scale)
        if inten.shape != (k_int.height, k_int.width) or depth.shape != inten.shape:
            raise _dimension_error(sensor, ts, inten.shape)
        pyr = build_pyramid(inten, depth, k_int, scales, normal_cfg)
        nodes.append(FrameNode(k, pose, pyr, float(ts), sensor.sensor_id))
    return nodes


def _load_sensor_device(dataset_dir, sensor, trajectory, scales, normal_cfg, device, threads):
    import torch

    from . import native as N
    from .pyramid_device import build_pyramids_device

    lib = N.load()
    k_int = sensor.intrinsics
    H, W = k_int.height, k_int.width
    n = len(trajectory)
    paths = [_frame_paths(dataset_dir, sensor, ts) for ts in trajectory.timestamps]

    def fetch(k):
        ipath, dpath = paths[k]
        wi, hi, bi, pi = _read_payload(ipath)
        wd, hd, bd, pd = _read_payload(dpath)
        ts = trajectory.timestamps[k]
        if (hi, wi) != (H, W) or (hd, wd) != (hi, wi):
            raise _dimension_error(sensor, ts, (hi, wi))
        if bd != 2:
            raise DatasetError(f"{dpath}: depth rasters must be 16-bit")
        return bi, pi, pd

    with ThreadPoolExecutor(max_workers=max(1, threads)) as pool:
        parts = list(pool.map(fetch, range(n)))
    kinds = {bi for bi, _, _ in parts}
    npx = H * W
    # one pinned staging buffer: intensity payloads (2 or 1 B/px), then depth
    ibytes = sum(len(pi) for _, pi, _ in parts)
    stage = torch.empty(ibytes + 2 * npx * n, dtype=torch.uint8, pin_memory=True)
    view = stage.numpy()
    off = 0
    for _, pi, _ in parts:
        view[off: off + len(pi)] = np.frombuffer(pi, dtype=np.uint8)
        off += len(pi)
    for _, _, pd in parts:
        view[off: off + len(pd)] = np.frombuffer(pd, dtype=np.uint8)
        off += len(pd)
    dev = torch.device(device)
    raw = stage.to(dev, non_blocking=True)
    inten = torch.empty((n, H, W), dtype=torch.float64, device=dev)
    depth = torch.empty((n, H, W), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    if len(kinds) == 1:
        kind = N.PBA_RASTER_U16_INTENSITY if kinds == {2} else N.PBA_RASTER_U8_INTENSITY
        N.check(lib.pba_decode_raster(raw.data_ptr(), n * npx, kind, 0.0, inten.data_ptr(),
                                      stream), "pba_decode_raster")
    else:  # mixed 8/16-bit intensity files: one launch per frame
        off = 0
        for k, (bi, pi, _) in enumerate(parts):
            kind = N.PBA_RASTER_U16_INTENSITY if bi == 2 else N.PBA_RASTER_U8_INTENSITY
            N.check(lib.pba_decode_raster(raw.data_ptr() + off, npx, kind, 0.0,
                                          inten[k].data_ptr(), stream), "pba_decode_raster")
            off += len(pi)
    N.check(lib.pba_decode_raster(raw.data_ptr() + ibytes, n * npx, N.PBA_RASTER_U16_DEPTH,
                                  float(sensor.depth_scale), depth.data_ptr(), stream),
            "pba_decode_raster")
    pyrs = build_pyramids_device(inten, depth, k_int, scales, normal_cfg, dev)
    return [FrameNode(k, pose, pyrs[k], float(ts), sensor.sensor_id)
            for k, (ts, pose) in enumerate(zip(trajectory.timestamps, trajectory.poses))]


def load_dataset(dataset_dir, scales=None, normal_cfg: NormalConfig | None = None, device=None,
                 threads: int = 8):
    """Dataset directory -> (manifest, trajectory, {sensor_id: [FrameNode]})
    (dataset_io.py:305-342).  Every trajectory row needs an intensity and a
    depth raster per sensor; pyramids are built on load — on the host
    (reference-exact) by default, or on the GPU with `device`."""
    dataset_dir = Path(dataset_dir)
    manifest = load_manifest(dataset_dir / "manifest")
    trajectory = load_trajectory(dataset_dir / manifest.trajectory_file)
    use_scales = scales or manifest.pyramid_scales
    frames = {}
    for sensor in manifest.sensors:
        if device is None:
            frames[sensor.sensor_id] = _load_sensor_host(dataset_dir, sensor, trajectory,
                                                         use_scales, normal_cfg)
        else:
            frames[sensor.sensor_id] = _load_sensor_device(dataset_dir, sensor, trajectory,
                                                           use_scales, normal_cfg, device, threads)
    return manifest, trajectory, frames


def write_dataset(dataset_dir, manifest: DatasetManifest, trajectory: Trajectory,
                  frames: dict) -> None:
    """Write a dataset directory: manifest, trajectory and, per sensor, the
    (intensity, depth_meters) arrays of every trajectory row in `frames`
    ({sensor_id: [(intensity, depth), ...]}).  The inverse of load_dataset
    (the reference writes the same layout from synthetic.generate_synthetic)."""
    dataset_dir = Path(dataset_dir)
    dataset_dir.mkdir(parents=True, exist_ok=True)
    save_manifest(manifest, dataset_dir / "manifest")
    save_trajectory(trajectory, dataset_dir / manifest.trajectory_file)
    for sensor in manifest.sensors:
        (dataset_dir / sensor.intensity_dir).mkdir(parents=True, exist_ok=True)
        (dataset_dir / sensor.depth_dir).mkdir(parents=True, exist_ok=True)
        for ts, (inten, depth) in zip(trajectory.timestamps, frames[sensor.sensor_id]):
            name = timestamp_name(ts) + ".pgm"
            write_intensity(dataset_dir / sensor.intensity_dir / name, inten)
            write_depth(dataset_dir / sensor.depth_dir / name, depth, sensor.depth_scale)


__all__ = [
    "DatasetError", "ManifestError", "MissingFileError", "DimensionMismatchError",
    "TrajectoryFormatError", "Trajectory", "trajectory_from_poses", "write_raster",
    "read_raster", "write_intensity", "read_intensity", "write_depth", "read_depth",
    "save_trajectory", "load_trajectory", "SensorConfig", "DatasetManifest", "save_manifest",
    "load_manifest", "timestamp_name", "load_dataset", "write_dataset",
]
