"""B200-native GWTF microbatch-routing min-cost-flow solver (arxiv 2509.21221).

The product is libgwtf.so (C-ABI in include/gwtf.h, sm_100a kernels in csrc/); this package is
its thin Python binding plus the multi-GPU sharding helper (dist.py).  See DESIGN.md.
"""
from ._lib import GWTF_HOST_PTRS, OBJ_MINIMAX, OBJ_SUM, GwtfError, lib  # noqa: F401
from .flow import ABSENT, Flow, RoundsResult, SolveResult, eq1_cost_tiles  # noqa: F401
from . import addition  # noqa: F401,E402
from . import multisource  # noqa: F401,E402
