"""B200-native (sm_100a) hot path of the hierarchical random walker, arXiv 2103.09564.

The product is the C-ABI library ``librw.so`` (include/rw.h) built from ``csrc/``;
``api`` is a thin ctypes binding (argument marshalling only).  No CPU fallback exists:
importing ``api`` works without a GPU, calling a compute function needs the CUDA build.
"""
from . import api  # noqa: F401
from .api import (  # noqa: F401
    brick_weights, brick_weights_ex, solve_bricks, solve_bricks_host, solve_labels, build_pyramid, build_pyramid_slab, Queue,
    solve_workspace_bytes, solve_labels_workspace_bytes, level_dims, set_solver, get_solver,
    solver, resident_available, hier_segment, hier_segment_labels, hier_segment_ooc, hier_segment_labels_ooc, pinned_empty, host_register, hier_ooc_alloc, stream_passes,
    set_stream_passes, get_stream_passes, set_resident_wide, get_resident_wide,
    set_device_loop, get_device_loop, device_loop, set_stream_zc, get_stream_zc, stream_zc,
    set_l2_workers, get_l2_workers, l2_workers,
)
