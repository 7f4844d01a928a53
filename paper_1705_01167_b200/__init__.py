"""B200-native CDDT range method: batched 2D ray casting against an occupancy
grid, the fused beam sensor model and the particle-filter step, on sm_100a.

Drop-in for the reference's range-method path (rangelib::Cddt / RangeMethod /
sensor_update); see DESIGN.md and include/rl_cddt.h.
"""
from .rangelib import *  # noqa: F401,F403
from .rangelib import __all__ as _rl_all

__all__ = list(_rl_all)
