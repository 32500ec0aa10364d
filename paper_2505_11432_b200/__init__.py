"""B200-native (sm_100a) MegaScale-MoE layer hot path.

Product code: CUDA kernels in csrc/ behind the C ABI of include/moe_b200.h,
loaded from libmoe_b200.so. There is no CPU fallback: operators raise when
the library or a GPU is missing.
"""
from ._lib import DomainError, MoEError, MoETimeout, launch_count, launch_count_reset, lib  # noqa: F401
from . import routing, ops  # noqa: F401

__all__ = ["routing", "ops", "lib", "DomainError", "MoEError", "MoETimeout"]
