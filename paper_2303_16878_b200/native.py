"""ctypes binding of the C ABI in include/pba.h (libpba_b200.so).

This is the whole boundary between the Python host and the sm_100a
kernels: plain pointers (torch tensor data_ptr()s), sizes and a stream.
The library is built in-tree by `paper_2303_16878_b200._build`; importing
this module never falls back to anything else — if the library is missing
or fails to load, `load()` raises.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

from . import _build

PBA_OK = 0
PBA_ERR_ARG = 1
PBA_ERR_CUDA = 2
PBA_ERR_SINGULAR = 3
PBA_ERR_PERTURBATION = 4
PBA_RASTER_U8_INTENSITY = 0
PBA_RASTER_U16_INTENSITY = 1
PBA_RASTER_U16_DEPTH = 2
PBA_PINHOLE = 0
PBA_SPHERICAL = 1
PBA_SOLVE_REUSE_PLAN = 1
PBA_CFG_PINHOLE_DST = 1  # pba_config.flags: pinhole destinations present (K1 prefetch)
RECORD_DOUBLES = 92
NORMALS_RECHECK_DOUBLES = 10
PARTIAL_DOUBLES = 32
# device-resident LM level (pba_lm_*): state indices and error codes
LM_COST, LM_COUNT, LM_LAMBDA, LM_FACTOR, LM_REL_TOL, LM_LAMBDA_CEILING = 0, 1, 2, 3, 4, 5
LM_COST_FLOOR, LM_ITERATION, LM_MAX_ITERATIONS, LM_STOP, LM_ERROR = 6, 7, 8, 9, 10
LM_N_RECORDS, LM_ACCEPTED, LM_STATE_DOUBLES = 11, 12, 16
LM_ERR_UNDERCONSTRAINED, LM_ERR_PERTURBATION, LM_MAX_COPY, LM_RECORD_DOUBLES = 1, 2, 8, 6

# symbols declared in include/pba.h, in header order
EXPORTED = (
    "pba_texel_bytes", "pba_ray_table_doubles", "pba_version", "pba_last_error",
    "pba_build_checked",
    "pba_kernel_launches",
    "pba_build_texels_scratch_bytes", "pba_build_texels", "pba_build_texels_batch", "pba_plan_chunks", "pba_linearize_scratch_bytes", "pba_linearize",
    "pba_plan_assembly", "pba_assemble", "pba_assemble_bsr", "pba_sum_totals",
    "pba_solve_work_bytes", "pba_solve_dense", "pba_solve_dense_ex", "pba_solve_dense_bsr",
    "pba_pcg_work_bytes", "pba_solve_pcg", "pba_solve_pcg_ex", "pba_solve_pcg_bsr",
    "pba_apply_step",
    "pba_lm_loop_begin", "pba_lm_decide", "pba_lm_loop_end", "pba_lm_loop_launch",
    "pba_lm_loop_destroy",
    "pba_overlap_counts", "pba_normals_scratch_bytes",
    "pba_estimate_normals", "pba_downscale_cues", "pba_decode_raster", "pba_atan2_batch",
    "pba_diag_section_cycles", "pba_diag_lm_stamp",
)


class Camera(ctypes.Structure):
    _fields_ = [("model", ctypes.c_int32), ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("_pad", ctypes.c_int32), ("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("cx", ctypes.c_double), ("cy", ctypes.c_double), ("depth_min", ctypes.c_double),
                ("depth_max", ctypes.c_double)]


class Frame(ctypes.Structure):
    _fields_ = [("texels", ctypes.c_void_p), ("mask", ctypes.c_void_p),
                ("ray_table", ctypes.c_void_p), ("cam", Camera)]


class Pair(ctypes.Structure):
    _fields_ = [("pose_i", ctypes.c_int32), ("pose_j", ctypes.c_int32), ("src", ctypes.c_int32),
                ("dst", ctypes.c_int32), ("ext", ctypes.c_int32), ("n_chunks", ctypes.c_int32),
                ("occ_tol", ctypes.c_double)]


class Config(ctypes.Structure):
    _fields_ = [("huber_delta", ctypes.c_double * 3), ("omega", ctypes.c_double * 5),
                ("pixel_stride", ctypes.c_int32), ("flags", ctypes.c_int32)]


class NormalConfigC(ctypes.Structure):
    _fields_ = [("k_tau", ctypes.c_double), ("radius_min", ctypes.c_double),
                ("radius_max", ctypes.c_double), ("min_points", ctypes.c_double),
                ("degeneracy_ratio", ctypes.c_double)]


assert ctypes.sizeof(Camera) == 64 and ctypes.sizeof(Frame) == 88 and ctypes.sizeof(Pair) == 32

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_dbl = ctypes.c_double
_sz = ctypes.c_size_t

_SIGNATURES = {
    "pba_texel_bytes": (_sz, []),
    "pba_ray_table_doubles": (_sz, [ctypes.POINTER(Camera)]),
    "pba_version": (ctypes.c_char_p, []),
    "pba_last_error": (ctypes.c_char_p, []),
    "pba_build_checked": (_i32, []),
    "pba_kernel_launches": (ctypes.c_uint64, []),
    "pba_build_texels_scratch_bytes": (_sz, [ctypes.POINTER(Camera)]),
    "pba_build_texels": (ctypes.c_int, [ctypes.POINTER(Camera), _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pba_build_texels_batch": (ctypes.c_int, [ctypes.POINTER(Camera), _i32, _vp, _vp, _vp, _vp,
                                              _vp, _vp, _vp]),
    "pba_plan_chunks": (ctypes.c_int, [_vp, _i32, _vp, _i32, _i32, _vp, _vp,
                                       ctypes.POINTER(_i64)]),
    "pba_linearize_scratch_bytes": (_sz, [_i32, _i64]),
    "pba_linearize": (ctypes.c_int, [_vp, _vp, _i32, _vp, _i64, _vp, _i32, _vp, _vp,
                                     ctypes.POINTER(Config), _i32, _vp, _vp, _vp]),
    "pba_plan_assembly": (ctypes.c_int, [_vp, _i32, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp,
                                         ctypes.POINTER(_i32)]),
    "pba_assemble": (ctypes.c_int, [_vp, _i32, _i32, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp,
                                    _vp, _vp]),
    "pba_assemble_bsr": (ctypes.c_int, [_vp, _i32, _i32, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp,
                                        _vp, _vp, _vp]),
    "pba_sum_totals": (ctypes.c_int, [_vp, _i32, _vp, _vp]),
    "pba_solve_work_bytes": (_sz, [_i32]),
    "pba_solve_dense": (ctypes.c_int, [_vp, _vp, _i32, _dbl, _vp, _vp, _vp, _vp, _vp]),
    "pba_solve_dense_ex": (ctypes.c_int, [_vp, _vp, _i32, _dbl, _vp, _vp, _vp, _i32, _vp, _vp,
                                          _vp]),
    "pba_solve_dense_bsr": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i32, _dbl, _vp, _vp, _vp, _i32,
                                           _vp, _vp, _vp]),
    "pba_pcg_work_bytes": (_sz, [_i32]),
    "pba_solve_pcg_bsr": (ctypes.c_int, [_vp, _vp, _i32, _dbl, _vp, _vp, _vp, _vp, _i32, _dbl,
                                         _vp, _vp, _vp, _vp, _vp]),
    "pba_solve_pcg_ex": (ctypes.c_int, [_vp, _vp, _i32, _dbl, _vp, _vp, _vp, _i32, _dbl, _vp,
                                        _vp, _vp, _vp, _vp]),
    "pba_solve_pcg": (ctypes.c_int, [_vp, _vp, _i32, _dbl, _vp, _vp, _i32, _dbl, _vp, _vp, _vp,
                                     _vp, _vp]),
    "pba_apply_step": (ctypes.c_int, [_vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "pba_lm_loop_begin": (ctypes.c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_uint64)]),
    "pba_lm_decide": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_uint64, _vp, _vp,
                                     _vp, _i32, _vp]),
    "pba_lm_loop_end": (ctypes.c_int, [_vp]),
    "pba_lm_loop_launch": (ctypes.c_int, [_vp, _vp]),
    "pba_lm_loop_destroy": (None, [_vp]),
    "pba_atan2_batch": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp]),
    "pba_diag_section_cycles": (ctypes.c_int, [_vp, _vp, _i32]),
    "pba_diag_lm_stamp": (ctypes.c_int, [_vp, _vp, _i32, _vp]),
    "pba_overlap_counts": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _i32, _dbl, _vp, _vp]),
    "pba_normals_scratch_bytes": (_sz, [ctypes.POINTER(Camera), _i32]),
    "pba_estimate_normals": (ctypes.c_int, [ctypes.POINTER(Camera), _vp, _vp, _i32,
                                            ctypes.POINTER(NormalConfigC), _vp, _vp, _vp, _i32,
                                            _vp, _vp]),
    "pba_downscale_cues": (ctypes.c_int, [ctypes.POINTER(Camera), _dbl, _i32, _vp, _vp, _vp,
                                          _i32, _i32, _vp, _vp, _vp, _vp]),
    "pba_decode_raster": (ctypes.c_int, [_vp, _i64, _i32, _dbl, _vp, _vp]),
}

_lib = None


class NativeError(RuntimeError):
    """A CUDA / argument failure reported by libpba_b200."""


def _checked() -> bool:
    import os

    return os.environ.get("PBA_CHECKED") == "1"


def library_path() -> Path:
    import os

    override = os.environ.get("PBA_LIBRARY")  # A/B experiments: another build of the same ABI
    if override:
        return Path(override)
    return _build.LIB_CHECKED if _checked() else _build.LIB


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load libpba_b200.so (building it in-tree with nvcc if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not path.exists():
        if not build_if_missing:
            raise NativeError(f"{path} is missing; run paper_2303_16878_b200._build.build()")
        _build.build(checked=_checked())
    lib = ctypes.CDLL(str(path))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc == PBA_OK:
        return
    msg = load().pba_last_error().decode(errors="replace")
    if rc == PBA_ERR_ARG:
        raise ValueError(f"{what}: {msg}")
    raise NativeError(f"{what} failed (code {rc}): {msg}")
