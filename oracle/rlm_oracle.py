"""CPU oracle for RLM-sort (recurse-last multiway mergesort) — TEST
INFRASTRUCTURE ONLY.

Restates ``mlpsort.rlm.rlm_sort`` (rlm.py:86-132) with numpy arrays.  Like
``oracle/ams_oracle.py`` it is the *checker*: only ``tests/`` (and the
fixture generator ``oracle/make_rlm_goldens.py``) import it; the product
package never does.

Parity pin: ``tests/test_rlm_oracle.py`` checks this restatement against
golden fixtures produced by the real reference (``oracle/make_rlm_goldens.py``
→ ``tests/golden/rlm/cases.json``): per-PE outputs (key and origin hashes),
per-level cut matrices, member sizes and level reports.

What is restated, and how:

* ``Element`` order is ``(key, origin_pe, origin_pos)`` (core.py:19-43); with
  PE-major inputs that is ``(key, origin index)``.  Every PE array is kept
  sorted by that order (rlm.py:96-97 local sort, 113-115 merges of sorted
  runs — a merge of sorted runs is the sort of their union).
* ``_cut_points`` (rlm.py:53-83): part g of a group receives the elements
  of global ranks ``(target[g-1], target[g]]`` with targets ``part + (1 if
  g < rem)`` accumulated.  ``multiselect_many`` (multiselect.py:45-137) finds
  them by randomized quickselect, but its *result* is unique — identities
  are unique, so ``splits[pe]`` = how many of the PE's elements are among
  the ``t`` globally smallest — and is computed here from one lexsort of
  the group.  (The ledger charges of the selection rounds depend on the
  pivot draws and are not restated.)
* delivery (rlm.py:108-110): the same ``deliver`` schemes as AMS-sort, with
  stream ``{stream}/L{lv}-g{lo}/deliver`` — the planners of
  ``ams_oracle`` are reused.
* level reports (rlm.py:118-131).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import ams_oracle as O

U64 = np.uint64


@dataclass
class RlmGroupInfo:
    level: int
    group_lo: int
    sizes: list            # member sizes before the level
    targets: list          # accumulated part targets (r - 1 of them)
    cuts: np.ndarray       # (P, r + 1) cut positions in every member's sorted array
    new_sizes: list
    stats: dict = field(default_factory=dict)


@dataclass
class RlmResult:
    keys: np.ndarray
    origin: np.ndarray      # origin index (input position) of every output element
    vals: np.ndarray | None
    pe_sizes: list
    levels: list            # list[list[RlmGroupInfo]]
    reports: list


def level_plan_check(p: int, group_counts) -> None:
    """``LevelPlan.__post_init__`` (rlm.py:29-41), same messages."""
    group_counts = tuple(group_counts)
    if p < 1:
        raise ValueError("need at least one PE")
    remaining = p
    for r in group_counts:
        if r < 1 or remaining % r != 0:
            raise ValueError(f"group counts {group_counts} do not divide {p}")
        remaining //= r
    if remaining != 1:
        raise ValueError(f"group counts {group_counts} do not telescope {p} to 1")


def part_targets(n_g: int, r: int) -> list:
    """rlm.py:60-66."""
    part, rem = divmod(n_g, r)
    out, acc = [], 0
    for g in range(r - 1):
        acc += part + (1 if g < rem else 0)
        out.append(acc)
    return out


def cut_points(keys: np.ndarray, org: np.ndarray, sizes: list, r: int):
    """Cut matrix of one group (rlm.py:53-83): ``cuts[j, g]`` .. ``cuts[j,
    g + 1]`` is member j's piece for part g.  ``keys``/``org`` hold the
    members' arrays back to back, each sorted by (key, origin)."""
    P = len(sizes)
    n_g = int(sum(sizes))
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    targets = part_targets(n_g, r)
    cuts = np.zeros((P, r + 1), np.int64)
    cuts[:, r] = np.asarray(sizes, np.int64)
    if n_g:
        order = np.lexsort((org, keys))              # global (key, origin) order
        rank = np.empty(n_g, np.int64)
        rank[order] = np.arange(n_g, dtype=np.int64)  # 0-based global rank
        for g, t in enumerate(targets):
            for j in range(P):
                # the member's elements are in rank order: count those < t
                rj = rank[offs[j]:offs[j + 1]]
                cuts[j, g + 1] = int(np.searchsorted(rj, t, side="left"))
    return targets, cuts


def rlm_sort(keys: np.ndarray, pe_sizes: list, group_counts: tuple, scheme: str = "simple",
             master_seed: int = 0, stream: str = "root", vals: np.ndarray | None = None) -> RlmResult:
    keys = np.ascontiguousarray(keys, dtype=U64)
    p = len(pe_sizes)
    level_plan_check(p, group_counts)
    n = int(sum(pe_sizes))
    sizes = [int(s) for s in pe_sizes]
    org = np.arange(n, dtype=np.int64)
    buf = keys.copy()
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    for pe in range(p):                                # rlm.py:96-97
        s, e = int(offs[pe]), int(offs[pe + 1])
        o = np.lexsort((org[s:e], buf[s:e]))
        buf[s:e] = buf[s:e][o]
        org[s:e] = org[s:e][o]
    groups = [(0, p)]
    all_levels, reports = [], []
    for lv, r in enumerate(group_counts):
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        new_buf = np.empty_like(buf)
        new_org = np.empty_like(org)
        new_sizes = list(sizes)
        infos, next_groups = [], []
        for lo, cnt in groups:
            gs, ge = int(offs[lo]), int(offs[lo + cnt])
            gsz = sizes[lo:lo + cnt]
            targets, cuts = cut_points(buf[gs:ge], org[gs:ge], gsz, r)
            pieces = np.diff(cuts, axis=1)             # (P, r)
            goff = np.concatenate([[0], np.cumsum(gsz)]).astype(np.int64)
            # Simple layout E: pieces (j, g) source-major inside each part g.
            parts_k, parts_o = [], []
            for g in range(r):
                for j in range(cnt):
                    a, b = int(goff[j] + cuts[j, g]), int(goff[j] + cuts[j, g + 1])
                    parts_k.append(buf[gs + a:gs + b])
                    parts_o.append(org[gs + a:gs + b])
            ek = np.concatenate(parts_k) if parts_k else np.zeros(0, U64)
            eo = np.concatenate(parts_o) if parts_o else np.zeros(0, np.int64)
            sub = cnt // r
            level_stream = f"{stream}/L{lv}-g{lo}"
            if scheme == "simple":                     # delivery.py:151-180
                ns = []
                for g in range(r):
                    m = int(pieces[:, g].sum())
                    for t in range(sub):
                        ns.append((m * (t + 1)) // sub - (m * t) // sub)
                stats = O._exchange_stats(pieces, sub, list(range(cnt)))
            else:
                if scheme == "deterministic":
                    slices, ns = O.deterministic_plan(pieces, lo)
                elif scheme == "permuted":
                    slices, ns = O.permuted_plan(pieces, master_seed, level_stream)
                elif scheme == "randomized":
                    slices, ns = O.randomized_plan(pieces, master_seed, level_stream)
                else:
                    raise ValueError(f"unknown delivery scheme {scheme!r}")
                ek = O.deterministic_relayout(ek, pieces, slices, ns)
                eo = O.deterministic_relayout(eo, pieces, slices, ns)
                stats = O._deterministic_stats(pieces, slices)
            # merge_runs (rlm.py:113-115): every member sorted by (key, origin).
            moff = np.concatenate([[0], np.cumsum(ns)]).astype(np.int64)
            for m in range(cnt):
                s, e = int(moff[m]), int(moff[m + 1])
                o = np.lexsort((eo[s:e], ek[s:e]))
                ek[s:e] = ek[s:e][o]
                eo[s:e] = eo[s:e][o]
            new_buf[gs:ge] = ek
            new_org[gs:ge] = eo
            new_sizes[lo:lo + cnt] = ns
            infos.append(RlmGroupInfo(lv, lo, list(gsz), targets, cuts, list(ns), stats))
            step = cnt // r
            next_groups.extend((lo + i * step, step) for i in range(r))
        buf, org, sizes, groups = new_buf, new_org, new_sizes, next_groups
        all_levels.append(infos)
        rep = {"level": lv + 1, "r": r, "max_load": max(sizes), "min_load": min(sizes)}
        for key in ("max_words", "max_msgs", "max_sent_msgs", "max_recv_msgs"):
            rep[key] = max(i.stats[key] for i in infos)
        reports.append(rep)
    out_vals = None if vals is None else np.asarray(vals)[org]
    return RlmResult(buf, org, out_vals, sizes, all_levels, reports)
