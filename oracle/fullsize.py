"""Full-size CPU oracle of ``ams_sort(scheme="simple")`` — TEST INFRASTRUCTURE ONLY.

The same algorithm as :func:`oracle.ams_oracle.ams_sort` (which restates
ams.py:271-313 and is pinned against the reference's own outputs in
``tests/test_oracle.py``), reorganised so it runs at BASELINE's full sizes
(2^28 - 2^30 keys) on the GPU box's host in minutes and ~4 bytes of extra
memory per key per copy:

* classification (ams.py:201-211) and the histogram run per member segment
  (one PE's array, a few MiB), not over the whole group buffer;
* the group's new layout — the stable sort of the group buffer by
  ``(g(b), j, b)`` (SURVEY §8 layout contract step 5, delivery.py:151-180,
  simnet.py:324-325) — is assembled from each segment's stable sort by
  bucket (bucket ids < 2^16 take numpy's radix sort), so no n-element
  composite key or argsort is ever built;
* segments are processed by a thread pool (numpy releases the GIL in
  searchsorted / argsort / take).

It reuses the pinned pieces of ``ams_oracle`` unchanged: the seeded sample
streams (``sample_indices``, ams.py:157-175), ``classify`` (bisect_left under
the tie-broken order) and ``group_plan`` (ams.py:78-154).  ``tests/
test_oracle.py::test_fullsize_matches_oracle`` checks it against
``ams_oracle.ams_sort`` and the golden fixtures.  The product never imports
this module.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from oracle import ams_oracle as O

U64 = np.uint64


@dataclass
class GroupFacts:
    """What the GPU's level records are compared with, per group."""

    group_lo: int
    n_g: int
    bucket_count: int
    sample_size: int
    splitter_keys: np.ndarray
    hist: np.ndarray          # (P, br) int64
    boundaries: tuple
    loads: tuple
    new_sizes: list


@dataclass
class FullResult:
    keys: np.ndarray          # final buffer: per-PE sorted arrays, PE-major
    pe_sizes: list
    levels: list              # per level: list[GroupFacts]


def _pool(threads: int | None):
    return ThreadPoolExecutor(max_workers=threads or min(32, os.cpu_count() or 1))


def _level_group(buf, out, gs, sizes, r, b, a, master_seed, stream, lv, lo, pool):
    """One level of one group (ams.py:214-268) over ``buf[gs : gs + n_g]``;
    writes the group's new layout to ``out[gs : gs + n_g]``."""
    P = len(sizes)
    n_g = int(sum(sizes))
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    br = min(b * r, n_g + 1)                                   # ams.py:224
    target = min(n_g, max(br - 1, math.ceil(a * br)))          # ams.py:225
    base, extra = divmod(target, P)                            # ams.py:166
    s_pos = []
    for i in range(P):                                         # ams.py:168-174
        take = min(base + (1 if i < extra else 0), sizes[i])
        sid = f"{stream}/L{lv}-g{lo}/sample/pe{lo + i}"
        s_pos.extend(int(offs[i]) + t for t in O.sample_indices(master_seed, sid, sizes[i], take))
    s_pos = np.asarray(s_pos, dtype=np.int64)
    drawn = len(s_pos)
    br = min(br, drawn + 1)                                    # ams.py:228
    if br <= 1:
        sk, sp = np.zeros(0, U64), np.zeros(0, np.int64)
    else:                                                      # ams.py:178-198
        s_keys = buf[gs + s_pos]
        order = np.lexsort((s_pos, s_keys))
        ranks = np.asarray(sorted({(i * drawn) // br for i in range(1, br)}), dtype=np.int64)
        sk, sp = s_keys[order[ranks]], s_pos[order[ranks]]

    def seg(j):
        a0, a1 = gs + int(offs[j]), gs + int(offs[j + 1])
        keys = buf[a0:a1]
        pos = np.arange(int(offs[j]), int(offs[j + 1]), dtype=np.int64)
        bk = O.classify(keys, pos, sk, sp)                      # ams.py:201-211
        h = np.bincount(bk, minlength=br)[:br].astype(np.int64)
        bk16 = bk.astype(np.uint16) if br <= 65536 else bk
        order = np.argsort(bk16, kind="stable")
        out[a0:a1] = keys[order]                               # segment, stable by bucket
        return h

    hist = np.stack(list(pool.map(seg, range(P)))) if P else np.zeros((0, br), np.int64)
    plan = O.group_plan(hist.sum(axis=0), r)                   # ams.py:236-238
    bnd = np.asarray(plan.boundaries, dtype=np.int64)
    # Bucket starts inside each stably bucket-sorted segment.
    cum = np.concatenate([np.zeros((P, 1), np.int64), np.cumsum(hist, axis=1)], axis=1)
    # New group buffer E_0 || ... || E_{r-1}, E_g = concat_j segment j's run
    # of buckets [B_g, B_{g+1}) (receive order = source order).
    pieces = []
    for g in range(r):
        for j in range(P):
            c0, c1 = int(cum[j, bnd[g]]), int(cum[j, bnd[g + 1]])
            if c1 > c0:
                pieces.append((gs + int(offs[j]) + c0, c1 - c0))
    tmp = np.empty(n_g, dtype=buf.dtype)
    at = 0
    for src, ln in pieces:
        tmp[at:at + ln] = out[src:src + ln]
        at += ln
    out[gs:gs + n_g] = tmp
    sub = P // r
    new_sizes = []
    for g in range(r):                                         # delivery.py:78-80
        m = int(plan.loads[g])
        for t in range(sub):
            new_sizes.append((m * (t + 1)) // sub - (m * t) // sub)
    return GroupFacts(lo, n_g, br, drawn, sk, hist, plan.boundaries, plan.loads, new_sizes)


def ams_sort_fullsize(keys: np.ndarray, pe_sizes, group_counts, oversampling=None,
                      overpartition: int = 16, imbalance: float = 0.2, master_seed: int = 0,
                      stream: str = "root", threads: int | None = None,
                      final_sort: bool = True) -> FullResult:
    """ams_sort (ams.py:271-313), scheme "simple", keys only (uint64 in the
    order-mapped encoding).  Same results as ``ams_oracle.ams_sort``."""
    keys = np.ascontiguousarray(keys, dtype=U64)
    p = len(pe_sizes)
    if math.prod(group_counts) != p:                           # ams.py:61-65
        raise ValueError(f"group counts {group_counts} do not telescope {p} PEs")
    n = int(sum(pe_sizes))
    a = oversampling if oversampling is not None else O.default_oversampling(n)
    buf = keys.copy()
    out = np.empty_like(buf)
    sizes = [int(s) for s in pe_sizes]
    groups = [(0, p)]
    levels = []
    with _pool(threads) as pool:
        for lv, r in enumerate(group_counts):
            offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
            new_sizes = list(sizes)
            facts, nxt = [], []
            for lo, cnt in groups:
                f = _level_group(buf, out, int(offs[lo]), sizes[lo:lo + cnt], r, overpartition,
                                 a, master_seed, stream, lv, lo, pool)
                new_sizes[lo:lo + cnt] = f.new_sizes
                facts.append(f)
                step = cnt // r
                nxt.extend((lo + i * step, step) for i in range(r))
            buf, out = out, buf
            sizes, groups = new_sizes, nxt
            levels.append(facts)
        if final_sort:                                         # ams.py:310-312 (F6)
            offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)

            def fin(pe):
                buf[offs[pe]:offs[pe + 1]].sort(kind="stable")
            list(pool.map(fin, range(p)))
    return FullResult(buf, sizes, levels)


def compare_levels(gpu_levels, ref: FullResult) -> list[str]:
    """Differences between the device run's level records
    (``engine.LevelRecord``) and the full-size oracle's: per group the bucket
    count, sample size, plan boundaries and loads, the per-member histogram;
    per level the next member sizes.  Empty list = identical."""
    bad = []
    for lv, (rec, facts) in enumerate(zip(gpu_levels, ref.levels)):
        if len(facts) != len(rec.group_first):
            bad.append(f"L{lv}: {len(rec.group_first)} groups vs {len(facts)}")
            continue
        for gi, f in enumerate(facts):
            tag = f"L{lv} g{f.group_lo}"
            if int(rec.group_first[gi]) != f.group_lo:
                bad.append(f"{tag}: first PE {int(rec.group_first[gi])}")
            if int(rec.bucket_count[gi]) != f.bucket_count:
                bad.append(f"{tag}: buckets {int(rec.bucket_count[gi])} vs {f.bucket_count}")
            if int(rec.sample_size[gi]) != f.sample_size:
                bad.append(f"{tag}: sample {int(rec.sample_size[gi])} vs {f.sample_size}")
            if tuple(int(x) for x in rec.boundaries[gi]) != tuple(f.boundaries):
                bad.append(f"{tag}: boundaries differ")
            if tuple(int(x) for x in rec.loads[gi]) != tuple(f.loads):
                bad.append(f"{tag}: loads differ")
            P = f.hist.shape[0]
            h = np.asarray(rec.seg_hist)[f.group_lo:f.group_lo + P, :f.bucket_count].astype(np.int64)
            if not np.array_equal(h, f.hist):
                bad.append(f"{tag}: histogram differs")
        mine = [int(x) for x in rec.new_sizes]
        theirs = [int(x) for f in facts for x in f.new_sizes]
        if mine != theirs:
            bad.append(f"L{lv}: next member sizes differ")
    return bad
