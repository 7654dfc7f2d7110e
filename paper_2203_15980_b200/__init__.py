"""delta-b200: a B200-native DELTA runtime (arXiv 2203.15980).

Plans tensor eviction/offload/recompute with the reference's exact policy on
its logical clock (libdelta, C++), then executes the plan on the GPU: an HBM
activation arena, copy-engine swap streams and sm_100a recompute kernels.
"""
from . import planner  # noqa: F401  (loads libdelta.so; raises if unbuilt)

__all__ = ["planner"]
