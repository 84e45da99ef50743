"""RLM-sort (recurse-last multiway mergesort) on the B200 path — drop-in for
the reference's ``mlpsort.rlm`` (rlm.py:22-132).

* :class:`LevelPlan` — same fields and ``ValueError`` texts as rlm.py:22-45.
* :func:`rlm_sort` — ``rlm_sort(net, data, plan, scheme, seed)`` with the
  reference's return structure ``(dict[pe] -> sorted list of Elements,
  level_reports)`` (rlm.py:86-132).
* :func:`rlm_sort_tensors` — the same sort over a device tensor of keys.

All per-element work runs in ``libams_b200.so`` (``ams_rlm_sort_run``): local
sorts, the exact multisequence selection of the cut positions (the unique
result of ``multiselect_many``, multiselect.py:45-137), the delivery relayout
and the merges.  The simulated network's ledger is not charged on this path
(the selection's charges depend on its pivot draws).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .engine import SCHEMES, check_out, key_kind_of
from .params import as_seed


@dataclass(frozen=True)
class LevelPlan:
    """Group counts per recursion level (rlm.py:22-45)."""

    p: int
    group_counts: tuple

    def __post_init__(self):
        object.__setattr__(self, "group_counts", tuple(int(r) for r in self.group_counts))
        if self.p < 1:
            raise ValueError("need at least one PE")
        remaining = self.p
        for r in self.group_counts:
            if r < 1 or remaining % r != 0:
                raise ValueError(f"group counts {self.group_counts} do not divide {self.p}")
            remaining //= r
        if remaining != 1:
            raise ValueError(f"group counts {self.group_counts} do not telescope {self.p} to 1")

    @property
    def levels(self) -> int:
        return len(self.group_counts)


@dataclass
class RlmOutput:
    keys: torch.Tensor
    origin: torch.Tensor          # input index of every output element
    vals: torch.Tensor | None
    pe_sizes: np.ndarray
    reports: list                 # rlm.py:118-131 dicts
    levels: list                  # per level: group_first / group_npe / sizes_before / cuts / new_sizes / stats
    launches: int


def _report(r) -> dict:
    return {"level": int(r.level), "r": int(r.r), "max_load": int(r.max_load),
            "min_load": int(r.min_load), "max_words": int(r.max_words), "max_msgs": int(r.max_msgs),
            "max_sent_msgs": int(r.max_sent_msgs), "max_recv_msgs": int(r.max_recv_msgs)}


def rlm_sort_tensors(keys: torch.Tensor, pe_sizes, plan, seed, vals: torch.Tensor | None = None,
                     scheme: str = "simple", key_kind=None) -> RlmOutput:
    """Sort device keys laid out PE-major (``pe_sizes``) as rlm_sort orders
    them; every PE ends with floor(n/p) or ceil(n/p)-balanced parts."""
    from .api import get_sorter
    if scheme not in SCHEMES:
        raise ValueError(f"unknown delivery scheme {scheme!r}; supported: {tuple(SCHEMES)}")
    if not isinstance(plan, LevelPlan):
        plan = LevelPlan(int(plan.p), tuple(plan.group_counts))
    if keys.dim() != 1 or not keys.is_cuda:
        raise ValueError("keys must be a 1-D CUDA tensor")
    sizes = np.asarray(pe_sizes, dtype=np.uint64)
    if len(sizes) != plan.p:
        raise ValueError("plan does not match the machine size")            # rlm.py:92-93
    n = int(sizes.sum())
    if n != keys.numel():
        raise ValueError(f"pe_sizes sum to {n}, keys has {keys.numel()} elements")
    if vals is not None and (vals.numel() != n or vals.element_size() != 8 or not vals.is_cuda
                             or vals.device != keys.device):
        raise ValueError("vals must be a CUDA tensor of n 8-byte values on the keys' device")
    kind = key_kind_of(keys, key_kind)
    master, stream_id = as_seed(seed)
    sorter = get_sorter(keys.device)
    keys = keys.contiguous()
    out = torch.empty_like(keys)
    origin = torch.empty(n, dtype=torch.int64, device=keys.device)
    out_vals = None
    if vals is not None:
        vals = vals.contiguous()
        out_vals = torch.empty_like(vals)
    check_out(out, n, keys.device, "out")
    ctx = sorter.ctx
    ctx.set_stream(torch.cuda.current_stream(keys.device).cuda_stream)
    launches0 = ctx.launches
    final_sizes, reps = ctx.rlm_sort_run(plan.group_counts, SCHEMES[scheme], master, stream_id, kind, sizes,
                                         keys if n else None, vals if n else None, out if n else None,
                                         origin if n else None, out_vals if n else None)
    levels = [ctx.rlm_level(lv) for lv in range(plan.levels)]
    return RlmOutput(out, origin, out_vals, final_sizes, [_report(r) for r in reps], levels,
                     ctx.launches - launches0)


def rlm_sort(net, data, plan, scheme: str, seed):
    """Drop-in for ``mlpsort.rlm.rlm_sort`` (rlm.py:86-132): per-PE sorted
    Element lists and one stats record per level.  Elements keep their
    identity; origin tags must increase along the PE-major input (as
    ``generate_input`` produces, bench.py:176)."""
    from .api import _flatten
    if not isinstance(plan, LevelPlan):
        plan = LevelPlan(int(plan.p), tuple(plan.group_counts))
    if plan.p != int(net.p):
        raise ValueError("plan does not match the machine size")
    p = plan.p
    flat, sizes = _flatten(data, p)
    n = len(flat)
    kind = "u64"
    keys = np.zeros(0, dtype=np.uint64)
    if n:
        tags = np.array([(e.origin_pe, e.origin_pos) for e in flat], dtype=np.int64)
        if n > 1:
            d0, d1 = np.diff(tags[:, 0]), np.diff(tags[:, 1])
            if np.any((d0 < 0) | ((d0 == 0) & (d1 <= 0))):
                raise ValueError("element origin tags must increase along the PE-major input "
                                 "order for the B200 path (tie-break by origin)")
        ks = [int(e.key) for e in flat]
        lo, hi = min(ks), max(ks)
        if lo < 0:
            if lo < -(1 << 63) or hi >= (1 << 63):
                raise ValueError("keys must fit in 64 bits")
            keys, kind = np.array(ks, dtype=np.int64), "i64"
        else:
            if hi >= (1 << 64):
                raise ValueError("keys must fit in 64 bits")
            keys = np.array(ks, dtype=np.uint64)
    dev = torch.device("cuda", torch.cuda.current_device())
    d_keys = torch.from_numpy(keys.view(np.int64)).to(dev)
    res = rlm_sort_tensors(d_keys, sizes, plan, seed, scheme=scheme, key_kind=kind)
    order = res.origin.cpu().numpy()
    out, start = {}, 0
    for pe in range(p):
        cnt = int(res.pe_sizes[pe])
        out[pe] = [flat[i] for i in order[start:start + cnt]]
        start += cnt
    return out, res.reports
