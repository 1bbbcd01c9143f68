"""B200-native (sm_100a) first-order immersed-boundary time step (arXiv math/0301321 §3.2).

The product is the C-ABI library libib_b200.so (include/ib.h); `ib` is its thin ctypes
binding.  See DESIGN.md.
"""
from .ib import (  # noqa: F401
    IBContext, IBError, load, library_path, EXPORTS,
    ib_create, ib_create3, ib_destroy, ib_set_stream, ib_set_option, ib_set_structure, ib_set_positions,
    ib_set_velocity, ib_set_drive, ib_set_fixed, ib_step, ib_get_fields, ib_get_positions, ib_get_step,
    ib_set_step, ib_stage_times, ib_launch_count,
    IB_OPT_PRESSURE, IB_OPT_STAGE_TIMING, IB_OPT_GRAPH,
)
