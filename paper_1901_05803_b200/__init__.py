"""B200-native execution of the resource-aware layer-placement (RALP) training step.

The planner surface (`profile`, `find_split`, `volume_ralp`, `JobSpec`, ...)
mirrors the reference `ralp` package (pkg/src/ralp/__init__.py); the training
step itself runs in libralpb200.so (hand-written sm_100a kernels) driven
through the C ABI in include/ralpb.h.
"""
from .planner import *  # noqa: F401,F403
from .planner import __dict__ as _planner_ns

__version__ = "0.1.0"
