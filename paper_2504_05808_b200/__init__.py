"""fastrs-b200: B200-native (sm_100a) local-thickness sphericity & roundness (arXiv 2504.05808).

Public API (torch CUDA tensors in, torch tensors out; all compute in libfastrs.so):
    edt_sq, local_thickness, sphericity_roundness, sphericity_roundness_host,
    diagnostics, profile, profile_read, spheroid_area, ramanujan_perimeter,
    sphericity_3d, sphericity_2d, release, touches_edge, filter_objects
"""
from .fastrs import (ASYNC, BORDER_BACKGROUND, DETERMINISTIC, FORCE_FALLBACK, HOST_IO, STAGES, FastrsError, diagnostics,
                     edt_sq, last_workspace, load, local_thickness, profile, profile_read, ramanujan_perimeter,
                     release, sphericity_2d, sphericity_3d, sphericity_roundness, sphericity_roundness_host,
                     spheroid_area, filter_objects, touches_edge, workspace, workspace_bytes)

__all__ = [
    "ASYNC", "BORDER_BACKGROUND", "DETERMINISTIC", "FORCE_FALLBACK", "HOST_IO", "STAGES", "FastrsError", "diagnostics", "edt_sq",
    "last_workspace", "load", "local_thickness", "profile", "profile_read", "ramanujan_perimeter", "release",
    "sphericity_2d", "sphericity_3d", "sphericity_roundness", "sphericity_roundness_host", "spheroid_area",
    "workspace", "workspace_bytes", "touches_edge", "filter_objects",
]
