"""B200-native AMS-sort (arXiv 1410.6754) — drop-in for the reference's
``mlpsort.ams.ams_sort`` hot path.

Host orchestration in Python; every per-element step runs in hand-written
sm_100a kernels of ``libams_b200.so`` (C ABI: include/ams_b200.h).
"""

from .params import AmsParams, Element, GroupPlan, SeedSpec  # noqa: F401

__all__ = ["AmsParams", "Element", "GroupPlan", "SeedSpec", "ams_sort", "ams_sort_tensors",
           "ams_sort_host", "AmsSorter", "LevelPlan", "rlm_sort", "rlm_sort_tensors"]


def __getattr__(name):
    # The CUDA-backed entry points load libams_b200.so on first use.
    if name in ("ams_sort", "ams_sort_tensors", "ams_sort_host"):
        from . import api
        return getattr(api, name)
    if name in ("LevelPlan", "rlm_sort", "rlm_sort_tensors"):
        from . import rlm
        return getattr(rlm, name)
    if name == "AmsSorter":
        from .engine import AmsSorter
        return AmsSorter
    raise AttributeError(name)
