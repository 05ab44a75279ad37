"""B200-native photometric bundle adjustment (arXiv 2303.16878 hot path).

Drop-in for the BA entry points and data types of the reference package
`photoba` (pkg/src/photoba/__init__.py:9-71): the same names, arguments and
results, with the per-iteration work — warp, residuals and Jacobians, the
12x12 JᵀWJ / JᵀWe accumulation, dense assembly, the damped linear solve and
the pose update — executed by hand-written sm_100a kernels
(csrc/*.cu, C ABI in include/pba.h).
"""

from .se3 import (InvalidPerturbationError, PerturbationVector, Pose, boxplus, exp, relative,
                  rotation_angle, skew)
from .camera import (PINHOLE, SPHERICAL, Intrinsics, SensorExtrinsics, project,
                     projective_jacobian, unproject)
from .cueimage import (CueImage, CuePyramid, DeviceCueImage, NormalConfig, PyramidConfigError,
                       build_cue_image, build_pyramid, estimate_normals, footprint_index,
                       sample)
from .pyramid_device import build_pyramids_device, estimate_normals_device
from .evaluation import (AteReport, DegenerateAlignmentError, NoAssociationError, associate,
                         ate_rmse, evaluate_ate, horn_align)
from .dataset import (DatasetError, DatasetManifest, DimensionMismatchError, ManifestError,
                      MissingFileError, SensorConfig, Trajectory, TrajectoryFormatError,
                      load_dataset, load_manifest, load_trajectory, read_depth, read_intensity,
                      read_raster, save_manifest, save_trajectory, timestamp_name,
                      trajectory_from_poses, write_dataset, write_depth, write_intensity,
                      write_raster)
from .pairgraph import (COVISIBILITY, ODOMETRY, Edge, FrameNode, GraphConfigError, MatchCriteria,
                        MatchGraph, build_graph, dump_edges, overlap_ratio)
from .bundle import (CONSECUTIVE, COUPLED, BAProblem, FusionConfigError, IterationRecord,
                     SolveResult, SolverConfig, UnderConstrainedError, check_connectivity,
                     reproject, solve_fusion, solve_hierarchical, solve_level, total_error)

__version__ = "0.1.0"

__all__ = [
    "AteReport", "DegenerateAlignmentError", "NoAssociationError", "associate", "ate_rmse",
    "evaluate_ate", "horn_align",
    "DatasetError", "DatasetManifest", "DimensionMismatchError", "ManifestError",
    "MissingFileError", "SensorConfig", "Trajectory", "TrajectoryFormatError", "load_dataset",
    "load_manifest", "load_trajectory", "read_depth", "read_intensity", "read_raster",
    "save_manifest", "save_trajectory", "timestamp_name", "trajectory_from_poses",
    "write_dataset", "write_depth", "write_intensity", "write_raster",
    "BAProblem", "CONSECUTIVE", "COUPLED", "COVISIBILITY", "CueImage", "CuePyramid",
    "DeviceCueImage", "Edge", "FrameNode", "FusionConfigError", "GraphConfigError",
    "InvalidPerturbationError", "Intrinsics", "IterationRecord", "MatchCriteria", "MatchGraph",
    "NormalConfig", "ODOMETRY", "PINHOLE", "PerturbationVector", "Pose", "PyramidConfigError", "SPHERICAL",
    "SensorExtrinsics", "SolveResult", "SolverConfig", "UnderConstrainedError", "boxplus",
    "build_cue_image", "build_graph", "build_pyramid", "build_pyramids_device", "check_connectivity", "dump_edges", "estimate_normals", "estimate_normals_device", "exp", "footprint_index",
    "overlap_ratio", "project", "projective_jacobian", "relative", "reproject", "rotation_angle",
    "sample", "skew",
    "solve_fusion", "solve_hierarchical", "solve_level", "total_error", "unproject",
]
