"""paper_2603_28160_b200 — B200-native FSM surface-topography hot path.

Drop-in for the reference package `millsurf` (arXiv 2603.28160) on its hot
path: the forward-solution-method sweep of cutting-edge points into a
min-height Z-map, the roughness indicators over it, and a batched
many-parameter-set mode. Same names, argument meaning and error types as
millsurf/__init__.py:46-92 for everything on that path; the sweep and the
reductions run as hand-written sm_100a CUDA kernels in libmsurf.so
(include/msurf.h). Host planning is NumPy; there is no CPU fallback.
"""

from .errors import ConfigError, DomainError, MillsurfError, NativeUnavailableError, SurfaceFormatError
from .geometry import (CuttingEdgePoint, EdgeDiscretization, ToolDefinition, default_point_count,
                       discretize_edge, edge_point, effective_half_length)
from .kinematics import (ProcessParameters, WorkpiecePoint, compose_transforms, derive_kinematics,
                         edge_to_tool_transform, spindle_to_workpiece_transform, tool_to_spindle_transform,
                         tooth_angle, transform_point)
from .grid import GridSpec, HeightField, TrajectoryRecord, locate, record_trajectory, update_min
from .extensions import Extensions
from .engine import (BenchmarkReport, BenchmarkRow, SimulationConfig, SimulationResult, run_benchmark,
                     simulate, simulate_batch, simulate_reference, time_step)
from .roughness import (ArealMetrics, LineProfile, ProfileRoughness, areal_metrics, areal_metrics_batch,
                        extract_profile, line_roughness, profile_roughness)
from .dataset import DatasetManifest, ParameterRange, generate_batch, generate_dataset, lhs_sample, uniform_sample
from .config import ConfigDocument, config_from_dict, parse_config, serialize_config
from .surface_io import export_views, read_surface, write_surface

__version__ = "0.1.0"

__all__ = [
    "ArealMetrics", "BenchmarkReport", "BenchmarkRow", "ConfigDocument", "ConfigError", "CuttingEdgePoint",
    "DatasetManifest", "DomainError", "config_from_dict", "export_views", "generate_dataset", "parse_config",
    "read_surface", "serialize_config", "write_surface",
    "EdgeDiscretization", "Extensions", "GridSpec", "HeightField", "LineProfile", "MillsurfError",
    "NativeUnavailableError", "ParameterRange", "ProcessParameters", "ProfileRoughness",
    "SimulationConfig", "SimulationResult", "SurfaceFormatError", "ToolDefinition", "TrajectoryRecord",
    "WorkpiecePoint", "areal_metrics", "areal_metrics_batch", "compose_transforms", "default_point_count",
    "derive_kinematics", "discretize_edge", "edge_point", "edge_to_tool_transform", "effective_half_length",
    "extract_profile", "generate_batch", "lhs_sample", "line_roughness", "locate", "profile_roughness",
    "record_trajectory", "run_benchmark", "simulate", "simulate_batch", "simulate_reference",
    "spindle_to_workpiece_transform", "time_step", "tool_to_spindle_transform", "tooth_angle",
    "transform_point", "uniform_sample", "update_min",
]
