"""B200-native connected-components labeling of 2D binary images by
block-parallel union-find in three kernels (arxiv 1708.08180): local merge with
coarse labeling, boundary analysis, link.

    import torch, paper_1708_08180_b200 as ccl
    labels = ccl.label(img_u8_cuda, connectivity=8)   # [H,W] or [B,H,W] -> int32

Output: 0 for background, 1 + the minimum raster index of the component for
foreground (per image).  The work runs in libccl.so (hand-written sm_100a
CUDA behind the C ABI in include/ccl.h); this package only marshals arguments.
"""
from ._binding import (  # noqa: F401
    CCLError,
    HostSession,
    HostPipeline,
    METHODS,
    MethodWorkspace,
    label_method,
    label_equal,
    label_3d,
    component_stats,
    STATS_FIELDS,
    StripLabeler,
    label_strips_emulated,
    strip_bounds,
    LIB_PATH,
    SIGNATURES,
    Workspace,
    boundary_work_items,
    default_tile_rows,
    strip_workspace_bytes,
    label,
    raw,
    stage_fns,
    stages,
    status_string,
    workspace_bytes,
)

__all__ = ["label", "label_method", "label_equal", "label_3d", "component_stats", "STATS_FIELDS", "MethodWorkspace", "METHODS", "Workspace", "StripLabeler", "label_strips_emulated", "strip_bounds", "HostSession", "HostPipeline", "CCLError", "workspace_bytes", "boundary_work_items", "default_tile_rows", "strip_workspace_bytes",
           "stages", "stage_fns", "status_string", "raw"]
