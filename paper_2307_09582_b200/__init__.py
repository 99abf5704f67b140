"""B200-native Guided Linear Upsampling (arXiv 2307.09582) hot path.

The product is the sm_100a CUDA library behind the C-ABI in include/glu_cuda.h
(paper_2307_09582_b200/lib/libglu_cuda.so) and the drop-in C++ API on top of it
(include/glu/*.hpp -> lib/libglu.so).  ``glu`` is the Python mirror of the
reference interface over device tensors; ``workloads`` builds the seeded
BASELINE.json inputs.
"""
from . import _native
from .glu import (  # noqa: F401
    GluConfig, GridSpec, JointResult, LargeErrorSet, Mode, ParamField, apply_field, error_map,
    find_large_error, grid_downsample, joint_optimize, mode_from_name, mode_name, neighborhood,
    op_color, op_matte, optimize_field, optimize_pixel_batch, optimize_pixel_exact,
    optimize_pixel_fast, optimize_pixel_gnu, optimize_pixels, pair_objective, self_error_map,
    solve_apply, trial_update_component, weight_exact, weight_fast,
)

__all__ = [n for n in dir() if not n.startswith("_")] + ["_native"]
