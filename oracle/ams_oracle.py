"""CPU oracle for the AMS-sort hot path — TEST INFRASTRUCTURE ONLY.

This module restates the reference algorithm (`mlpsort.ams.ams_sort` with
``scheme="simple"`` or ``"deterministic"``) with numpy arrays so the GPU path can be checked at
sizes the pure-Python reference cannot reach.  It is the *checker*: only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(`paper_1410_6754_b200`) never imports, links or executes anything here.

Parity pin: every function cites the reference file:line it restates, and
``tests/test_oracle.py`` checks this oracle against golden fixtures produced
by running the real reference (``oracle/make_goldens.py`` →
``tests/golden/*.json``).  Parity is therefore pinned against the reference
itself, not only against this restatement.

Element identity: the reference orders ``Element(key, origin_pe,
origin_pos)`` lexicographically (core.py:19-43).  Inside one PE group the
reference's concatenation keeps equal keys in origin order, so
``(key, position-in-group-buffer)`` is the same strict total order; the
oracle carries positions implicitly as array indices.
"""

from __future__ import annotations

import hashlib
import math
import random
from dataclasses import dataclass, field

import numpy as np

U64 = np.uint64


# --------------------------------------------------------------------------
# Seeded streams  (core.py:46-71)

def stream_seed_int(master_seed: int, stream_id: str) -> int:
    """``int.from_bytes(SeedSpec(master, stream)._digest(), "big")``
    (core.py:62-67): blake2b-128 of ``f"{master}\\x1f{stream}\\x1f"``."""
    text = f"{master_seed}\x1f{stream_id}\x1f"
    return int.from_bytes(
        hashlib.blake2b(text.encode(), digest_size=16).digest(), "big")


def sample_indices(master_seed: int, stream_id: str, n: int, take: int) -> list[int]:
    """``sorted(Random(seed).sample(range(n), take))`` (ams.py:171-173)."""
    rng = random.Random(stream_seed_int(master_seed, stream_id))
    return sorted(rng.sample(range(n), take))


# --------------------------------------------------------------------------
# Consecutive-bucket grouping  (ams.py:78-154)

@dataclass(frozen=True)
class Plan:
    boundaries: tuple
    loads: tuple
    max_load: int


def _scan(sizes, r, limit):
    """Greedy packing under ``limit`` (ams.py:78-109)."""
    overflow = None
    boundaries = [0]
    loads = []
    cur = 0
    for i, size in enumerate(sizes):
        if size > limit:
            return None, overflow
        if cur + size > limit:
            if overflow is None or cur + size < overflow:
                overflow = cur + size
            boundaries.append(i)
            loads.append(cur)
            cur = size
        else:
            cur += size
    boundaries.append(len(sizes))
    loads.append(cur)
    if len(loads) > r:
        return None, overflow
    while len(loads) < r:
        boundaries.append(len(sizes))
        loads.append(0)
    return Plan(tuple(boundaries), tuple(loads), max(loads)), overflow


def group_plan(sizes, r: int) -> Plan:
    """Binary search over the scan with overflow tightening
    (ams.py:119-154)."""
    sizes = [int(s) for s in sizes]
    total = sum(sizes)
    lo = max(max(sizes), -(-total // r))
    b_est = max(1, len(sizes) // r)
    hi = max(lo, math.ceil(total / r * (1.0 + 4.0 / b_est)))
    plan, overflow = _scan(sizes, r, hi)
    if plan is None:
        lo = max(lo, overflow if overflow is not None else hi + 1)
        hi = total
        plan, _ = _scan(sizes, r, hi)
    hi = plan.max_load
    best = plan
    while lo < hi:
        mid = (lo + hi) // 2
        plan, overflow = _scan(sizes, r, mid)
        if plan is not None:
            hi = plan.max_load
            best = plan
        else:
            lo = overflow if overflow is not None else mid + 1
    return best


# --------------------------------------------------------------------------
# One level of one group  (ams.py:214-268 + delivery.py:151-180)

@dataclass
class LevelInfo:
    """What the oracle records about one group at one level (for parity)."""

    level: int                 # 0-based lv as in ams.py:285
    group_lo: int              # first PE of the group
    n_g: int
    bucket_count: int
    sample_size: int
    splitter_keys: np.ndarray  # (br-1,) uint64
    splitter_pos: np.ndarray   # (br-1,) int64, position in group buffer
    hist: np.ndarray           # (P, br) per-member bucket histogram
    plan: Plan
    new_sizes: list            # sizes of the next-level member arrays
    stats: dict = field(default_factory=dict)


def classify(keys: np.ndarray, pos: np.ndarray, s_keys: np.ndarray,
             s_pos: np.ndarray) -> np.ndarray:
    """Bucket = number of splitters strictly below ``(key, pos)``
    (ams.py:201-211, bisect_left at 210)."""
    if len(s_keys) == 0:
        return np.zeros(len(keys), dtype=np.int64)
    b = np.searchsorted(s_keys, keys, side="left").astype(np.int64)
    hi = np.searchsorted(s_keys, keys, side="right")
    tie = np.nonzero(hi > b)[0]
    if len(tie):
        # Equal-key splitter runs: add the run members with a smaller
        # position (splitters are sorted by (key, pos)).
        for k in np.unique(keys[tie]):
            sel = tie[keys[tie] == k]
            lo_i = np.searchsorted(s_keys, k, side="left")
            hi_i = np.searchsorted(s_keys, k, side="right")
            b[sel] += np.searchsorted(s_pos[lo_i:hi_i], pos[sel], side="left")
    return b


def select_splitters(sample_keys, sample_pos, br):
    """Splitters = sorted sample at ranks ``(i*S)//br`` (ams.py:178-198;
    fastsort.py:57-130 ranks the same set)."""
    S = len(sample_keys)
    if br <= 1:
        return np.zeros(0, dtype=U64), np.zeros(0, dtype=np.int64)
    order = np.lexsort((sample_pos, sample_keys))
    ranks = sorted({(i * S) // br for i in range(1, br)})
    idx = order[np.asarray(ranks, dtype=np.int64)]
    return sample_keys[idx], sample_pos[idx]


def _exchange_stats(piece_sizes: np.ndarray, sub_sizes: int, members: list):
    """Data-exchange shape of ``deliver_simple`` (delivery.py:151-180,
    _slice_range 83-106) as ``Network.exchange`` counts it
    (simnet.py:294-335): self messages and empty payloads are free."""
    P, r = piece_sizes.shape
    sub = P // r
    sw = np.zeros(P, np.int64); rw = np.zeros(P, np.int64)
    sm = np.zeros(P, np.int64); rm = np.zeros(P, np.int64)
    for g in range(r):
        col = piece_sizes[:, g]
        m = int(col.sum())
        starts = np.concatenate([[0], np.cumsum(col)[:-1]])
        for j in range(P):
            size = int(col[j]); start = int(starts[j])
            if size == 0 or m == 0:
                continue
            for t in range(sub):
                lo = (m * t) // sub; hi = (m * (t + 1)) // sub
                take = min(start + size, hi) - max(start, lo)
                if take <= 0:
                    continue
                dest = g * sub + t
                if dest != j:
                    sw[j] += take; rw[dest] += take; sm[j] += 1; rm[dest] += 1
    hs, hr = int(sw.max(initial=0)), int(rw.max(initial=0))
    ms, mr = int(sm.max(initial=0)), int(rm.max(initial=0))
    return {"max_words": max(hs, hr), "max_msgs": max(ms, mr),
            "max_sent_msgs": ms, "max_recv_msgs": mr}


def key64(master_seed: int, stream_id: str, index: int) -> int:
    """``SeedSpec.key64`` (core.py:69-71): the first 8 bytes (big endian) of
    blake2b-128 of ``f"{master}\x1f{stream}\x1fk{index}"``."""
    text = f"{master_seed}\x1f{stream_id}\x1fk{index}"
    return int.from_bytes(hashlib.blake2b(text.encode(), digest_size=16).digest()[:8], "big")


def _mix64(x: int) -> int:
    """splitmix64 finalizer (core.py:74-79)."""
    m = 0xFFFFFFFFFFFFFFFF
    x &= m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


def feistel_order(n: int, master_seed: int, stream_id: str) -> list:
    """``sorted(range(n), key=feistel_new(n, seed).apply)`` (delivery.py:
    131-134; core.py:96-159): four keyed digit-pair rounds over the padded
    square domain side**2, cycle-walking values >= n."""
    side = math.isqrt(n)
    if side * side < n:
        side += 1
    tables = [[_mix64(b ^ key64(master_seed, stream_id, i)) % side for b in range(side)]
              for i in range(4)]

    def apply(i):
        x = i
        for _ in range(side * side):
            hi, lo = divmod(x, side)
            for t in tables:
                lo, hi = hi, (lo + t[hi]) % side
            x = lo + hi * side
            if x < n:
                return x
        raise RuntimeError("cycle walk failed to terminate; broken bijection")

    return sorted(range(n), key=apply)


def permuted_plan(piece_sizes: np.ndarray, master_seed: int, level_stream: str):
    """``deliver_simple_permuted`` (delivery.py:151-185): each subgroup g
    enumerates the sending members in the Feistel order of stream
    ``{level_stream}/deliver/order-g{g}``; member t owns numbers
    ``[m t / p', m (t+1) / p')`` of that enumeration.  Returns slices like
    :func:`deterministic_plan` and the new member sizes."""
    P, r = piece_sizes.shape
    if P % r != 0:
        raise ValueError(f"{P} PEs cannot form {r} groups")
    sub = P // r
    slices = {}
    new_sizes = [0] * P
    for g in range(r):
        order = feistel_order(P, master_seed, f"{level_stream}/deliver/order-g{g}")
        m = int(piece_sizes[:, g].sum())
        start = 0
        for j in order:
            size = int(piece_sizes[j, g])
            if size:
                cuts = []
                t = ((start + 1) * sub + m - 1) // m - 1          # _slice_range
                covered = 0
                while covered < size and t < sub:
                    hi = (m * (t + 1)) // sub
                    take = min(start + size, hi) - (start + covered)
                    if take > 0:
                        cuts.append((t, covered, take))
                        covered += take
                    t += 1
                slices[(j, g)] = cuts
            start += size
        for t in range(sub):
            new_sizes[g * sub + t] = (m * (t + 1)) // sub - (m * t) // sub
    return slices, new_sizes


def default_delegation_factor(p: int, r: int) -> int:
    """delivery.py:309-315."""
    if r * p <= 2:
        return 1
    a = 0.5 * (math.sqrt(1.0 + r / math.log(r * p / 2.0)) - 1.0)
    return max(1, math.floor(a))


def feistel_apply_all(n: int, master_seed: int, stream_id: str) -> list:
    """``[feistel_new(n, seed).apply(i) for i in range(n)]`` (core.py:96-159)."""
    order = feistel_order(n, master_seed, stream_id)
    perm = [0] * n
    for rank, i in enumerate(order):
        perm[i] = rank
    return perm


def randomized_plan(piece_sizes: np.ndarray, master_seed: int, level_stream: str):
    """``deliver_randomized`` (delivery.py:318-436) with the default
    delegation factor: pieces above s = ceil(a n / (r p)) are cut into
    s-element chunks (plus a remainder); full chunks are delegated to holder
    ``feistel(rank) % p`` (stream ``…/deliver/delegate``); subgroup g numbers
    the chunks holder by holder in the Feistel order of ``…/deliver/order-g{g}``,
    each holder's chunks in ``Random(…/deliver/reorder-g{g}-h{holder}).shuffle``
    order; members own quota slots of that numbering."""
    P, r = piece_sizes.shape
    if P % r != 0:
        raise ValueError(f"{P} PEs cannot form {r} groups")
    sub = P // r
    n = int(piece_sizes.sum())
    a = default_delegation_factor(P, r)
    s = max(1, -(-(a * n) // (r * P)))
    chunks = []
    for j in range(P):
        for g in range(r):
            size = int(piece_sizes[j, g])
            if size == 0:
                continue
            if size > s:
                whole, rem = divmod(size, s)
                for c in range(whole):
                    chunks.append((j, g, c * s, s, True))
                if rem:
                    chunks.append((j, g, whole * s, rem, False))
            else:
                chunks.append((j, g, 0, size, False))
    dstream = f"{level_stream}/deliver"
    large = [i for i, ch in enumerate(chunks) if ch[4]]
    holder_of = {}
    if large:
        perm = feistel_apply_all(len(large), master_seed, f"{dstream}/delegate")
        for rank, cid in enumerate(large):
            holder_of[cid] = perm[rank] % P
    held = {}
    for cid, (j, g, off, ln, lg) in enumerate(chunks):
        held.setdefault((g, holder_of.get(cid, j)), []).append(cid)
    start_of = {}
    totals = [0] * r
    for g in range(r):
        running = 0
        for holder in feistel_order(P, master_seed, f"{dstream}/order-g{g}"):
            mine = held.get((g, holder), [])
            if not mine:
                continue
            rng = random.Random(stream_seed_int(master_seed, f"{dstream}/reorder-g{g}-h{holder}"))
            rng.shuffle(mine)
            for cid in mine:
                start_of[cid] = running
                running += chunks[cid][3]
        totals[g] = running
    slices = {}
    for cid, (j, g, off, ln, lg) in enumerate(chunks):
        m, start = totals[g], start_of[cid]
        t = ((start + 1) * sub + m - 1) // m - 1               # _slice_range
        covered = 0
        while covered < ln and t < sub:
            hi = (m * (t + 1)) // sub
            take = min(start + ln, hi) - (start + covered)
            if take > 0:
                slices.setdefault((j, g), []).append((t, off + covered, take))
                covered += take
            t += 1
    for key in slices:
        slices[key].sort(key=lambda c: c[1])
    new_sizes = [0] * P
    for g in range(r):
        for t in range(sub):
            new_sizes[g * sub + t] = (totals[g] * (t + 1)) // sub - (totals[g] * t) // sub
    return slices, new_sizes


def deterministic_plan(piece_sizes: np.ndarray, group_lo: int = 0):
    """Member assignment of ``deliver_deterministic`` (delivery.py:188-306):
    small pieces (size * 2 * p * r <= n) go whole to member
    ``small_index // r`` of their subgroup; large pieces fill the members'
    residual quota capacity (delivery.py:78-80) by merging the two prefix
    sums, one member after another.  Returns ``slices[(j, g)] = [(t,
    offset, length), ...]`` (t = member of subgroup g) and the new member
    sizes (members in group order).  Raises ValueError for a piece above
    ceil(n/p) (delivery.py:212-217) and RuntimeError when the residual
    capacities cannot hold the large pieces (delivery.py:274-276)."""
    P, r = piece_sizes.shape
    if P % r != 0:
        raise ValueError(f"{P} PEs cannot form {r} groups")
    sub = P // r
    n = int(piece_sizes.sum())
    cap = -(-n // P)
    for j in range(P):
        for g in range(r):
            if int(piece_sizes[j, g]) > cap:
                raise ValueError(f"piece ({group_lo + j},{g}) larger than ceil(n/p): "
                                 f"{int(piece_sizes[j, g])} > {cap}")

    def is_small(size):
        return size * 2 * P * r <= n

    slices = {}
    for g in range(r):
        m_g = int(piece_sizes[:, g].sum())
        caps = [(m_g * (t + 1)) // sub - (m_g * t) // sub for t in range(sub)]
        small_load = [0] * sub
        small_index = 0
        larges = []
        for j in range(P):
            size = int(piece_sizes[j, g])
            if size == 0:
                continue
            if not is_small(size):
                larges.append((j, size))
                continue
            t = small_index // r
            small_index += 1
            small_load[t] += size
            slices[(j, g)] = [(t, 0, size)]
        bounds = [0]
        for t in range(sub):
            bounds.append(bounds[-1] + max(0, caps[t] - small_load[t]))
        pos = 0
        for j, size in larges:
            t = int(np.searchsorted(bounds, pos, side="right")) - 1   # bisect_right
            covered = 0
            cuts = []
            while covered < size:
                if t >= sub:
                    raise RuntimeError("residual capacities cannot hold the large pieces")
                take = min(pos + size, bounds[t + 1]) - (pos + covered)
                if take > 0:
                    cuts.append((t, covered, take))
                    covered += take
                t += 1
            slices[(j, g)] = cuts
            pos += size
    new_sizes = [0] * P
    for (j, g), cuts in slices.items():
        for t, _, ln in cuts:
            new_sizes[g * sub + t] += ln
    return slices, new_sizes


def _deterministic_stats(piece_sizes: np.ndarray, slices: dict):
    """Data-exchange shape of the deterministic delivery's data messages
    (``_execute``, delivery.py:109-120, counted by simnet.py:294-335)."""
    P, r = piece_sizes.shape
    sub = P // r
    sw = np.zeros(P, np.int64); rw = np.zeros(P, np.int64)
    sm = np.zeros(P, np.int64); rm = np.zeros(P, np.int64)
    for (j, g), cuts in slices.items():
        for t, _, ln in cuts:
            dest = g * sub + t
            if ln > 0 and dest != j:
                sw[j] += ln; rw[dest] += ln; sm[j] += 1; rm[dest] += 1
    hs, hr = int(sw.max(initial=0)), int(rw.max(initial=0))
    ms, mr = int(sm.max(initial=0)), int(rm.max(initial=0))
    return {"max_words": max(hs, hr), "max_msgs": max(ms, mr),
            "max_sent_msgs": ms, "max_recv_msgs": mr}


def deterministic_relayout(e_layout: np.ndarray, piece_sizes: np.ndarray, slices: dict,
                           new_sizes: list) -> np.ndarray:
    """Member arrays of the deterministic delivery from the simple group
    layout E (pieces (j, g) source-major inside each subgroup g): member
    (g, t) receives its slices in source order (inbox order, simnet.py:324-325)."""
    P, r = piece_sizes.shape
    sub = P // r
    g_start = np.concatenate([[0], np.cumsum(piece_sizes.sum(axis=0))]).astype(np.int64)
    p_start = np.zeros((P, r), np.int64)
    for g in range(r):
        p_start[:, g] = g_start[g] + np.concatenate([[0], np.cumsum(piece_sizes[:, g])[:-1]])
    out = np.empty_like(e_layout)
    at = 0
    for D in range(P):
        g, t = divmod(D, sub)
        for j in range(P):
            for tt, off, ln in slices.get((j, g), ()):
                if tt == t:
                    s0 = int(p_start[j, g]) + off
                    out[at:at + ln] = e_layout[s0:s0 + ln]
                    at += ln
    assert at == len(e_layout) and at == sum(new_sizes)
    return out


def ams_level(buf: np.ndarray, sizes: list, r: int, b: int, a: float,
              master_seed: int, stream: str, level: int, group_lo: int,
              vals: np.ndarray | None = None, with_stats: bool = False,
              scheme: str = "simple", org: np.ndarray | None = None):
    """One level on one group whose member arrays are consecutive in
    ``buf`` (ams.py:214-268).  Returns the new group buffer (the stable
    ``(g, j, b)`` order of SURVEY §8 layout contract, or the deterministic
    delivery's member arrays), new member sizes, a LevelInfo and the new
    origin tags.

    ``org`` = origin of every element (its index in the sort's input): the
    reference breaks key ties by ``(origin_pe, origin_pos)`` (core.py:19-43).
    Under "simple" delivery origin order equals group-buffer order (SURVEY
    F6); "deterministic" delivery can place a later source's piece in an
    earlier member, so ties are broken by the carried origin here."""
    P = len(sizes)
    n_g = int(sum(sizes))
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    br = min(b * r, n_g + 1)                                   # ams.py:224
    target = min(n_g, max(br - 1, math.ceil(a * br)))          # ams.py:225
    base, extra = divmod(target, P)                            # ams.py:166
    s_idx = []
    for i in range(P):                                         # ams.py:168-174
        quota = base + (1 if i < extra else 0)
        take = min(quota, sizes[i])
        pe = group_lo + i
        sid = f"{stream}/L{level}-g{group_lo}/sample/pe{pe}"
        idx = sample_indices(master_seed, sid, sizes[i], take)
        s_idx.extend(int(offs[i]) + t for t in idx)
    s_pos = np.asarray(s_idx, dtype=np.int64)
    drawn = len(s_pos)
    br = min(br, drawn + 1)                                    # ams.py:228
    if org is None:
        org = np.arange(n_g, dtype=np.int64)
    s_org = org[s_pos]
    if br <= 1:
        sk = np.zeros(0, dtype=U64); so = sp = np.zeros(0, dtype=np.int64)
    else:                                                      # ams.py:178-198
        order_s = np.lexsort((s_org, buf[s_pos]))
        ranks = sorted({(i * drawn) // br for i in range(1, br)})
        sel = order_s[np.asarray(ranks, dtype=np.int64)]
        sk, so, sp = buf[s_pos][sel], s_org[sel], s_pos[sel]
    bucket = classify(buf, org, sk, so)
    member = np.repeat(np.arange(P, dtype=np.int64), sizes)
    hist = np.zeros((P, br), dtype=np.int64)
    np.add.at(hist, (member, bucket), 1)
    plan = group_plan(hist.sum(axis=0), r)                     # ams.py:236-238
    bnd = np.asarray(plan.boundaries, dtype=np.int64)
    gid = np.searchsorted(bnd, bucket, side="right") - 1
    # Empty trailing groups share boundary == br; buckets never reach br.
    comp = (gid * P + member) * br + bucket
    order = np.argsort(comp, kind="stable")                    # F10 layout
    out = buf[order]
    out_vals = vals[order] if vals is not None else None
    out_org = org[order]
    sub = P // r
    pieces = np.zeros((P, r), np.int64)
    for g in range(r):
        pieces[:, g] = hist[:, bnd[g]:bnd[g + 1]].sum(axis=1)
    if scheme in ("deterministic", "permuted", "randomized"):  # delivery.py:151-436
        if scheme == "deterministic":
            slices, new_sizes = deterministic_plan(pieces, group_lo)
        elif scheme == "permuted":
            slices, new_sizes = permuted_plan(pieces, master_seed,
                                              f"{stream}/L{level}-g{group_lo}")
        else:
            slices, new_sizes = randomized_plan(pieces, master_seed,
                                                f"{stream}/L{level}-g{group_lo}")
        out = deterministic_relayout(out, pieces, slices, new_sizes)
        out_org = deterministic_relayout(out_org, pieces, slices, new_sizes)
        if out_vals is not None:
            out_vals = deterministic_relayout(out_vals, pieces, slices, new_sizes)
    elif scheme == "simple":
        new_sizes = []
        for g in range(r):                                     # delivery.py:78-80
            m = int(plan.loads[g])
            for t in range(sub):
                new_sizes.append((m * (t + 1)) // sub - (m * t) // sub)
    else:
        raise ValueError(f"unknown delivery scheme {scheme!r}")
    info = LevelInfo(level, group_lo, n_g, br, drawn, sk, sp, hist, plan,
                     new_sizes)
    if with_stats:
        if scheme in ("deterministic", "permuted", "randomized"):
            info.stats = _deterministic_stats(pieces, slices)
        else:
            info.stats = _exchange_stats(pieces, sub, list(range(P)))
    return out, out_vals, new_sizes, info, out_org


@dataclass
class SortResult:
    keys: np.ndarray
    vals: np.ndarray | None
    pe_sizes: list
    levels: list          # list[list[LevelInfo]] per level, per group
    reports: list         # reference-shaped level reports (ams.py:296-308)


def default_oversampling(n: int) -> float:
    """ams.py:278-280."""
    return 1.6 * math.log10(max(n, 10))


def ams_sort(keys: np.ndarray, pe_sizes: list, group_counts: tuple,
             oversampling: float | None = None, overpartition: int = 16,
             imbalance: float = 0.2, master_seed: int = 0,
             stream: str = "root", vals: np.ndarray | None = None,
             with_stats: bool = True, scheme: str = "simple") -> SortResult:
    """Restatement of ``ams_sort`` (ams.py:271-313) with ``scheme`` "simple"
    (delivery.py:151-180) or "deterministic" (delivery.py:188-306).
    ``keys`` is the PE-major concatenation of the per-PE inputs (uint64)."""
    keys = np.ascontiguousarray(keys, dtype=U64)
    p = len(pe_sizes)
    if math.prod(group_counts) != p:                           # ams.py:61-65
        raise ValueError(f"group counts {group_counts} do not telescope {p} PEs")
    n = int(sum(pe_sizes))
    a = oversampling if oversampling is not None else default_oversampling(n)
    k = len(group_counts)
    eps_l = (1.0 + imbalance) ** (1.0 / k) - 1.0               # ams.py:58-59
    buf = keys.copy()
    vbuf = None if vals is None else np.asarray(vals).copy()
    obuf = np.arange(n, dtype=np.int64)                        # origin tags
    sizes = [int(s) for s in pe_sizes]
    groups = [(0, p)]                                          # (lo, count)
    all_levels = []
    reports = []
    for lv, r in enumerate(group_counts):
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        new_buf = np.empty_like(buf)
        new_obuf = np.empty_like(obuf)
        new_vbuf = None if vbuf is None else np.empty_like(vbuf)
        new_sizes = list(sizes)
        infos = []
        next_groups = []
        for lo, cnt in groups:
            gs, ge = int(offs[lo]), int(offs[lo + cnt])
            out, out_v, ns, info, out_o = ams_level(
                buf[gs:ge], sizes[lo:lo + cnt], r, overpartition, a,
                master_seed, stream, lv, lo,
                None if vbuf is None else vbuf[gs:ge], with_stats, scheme, obuf[gs:ge])
            new_buf[gs:ge] = out
            new_obuf[gs:ge] = out_o
            if new_vbuf is not None:
                new_vbuf[gs:ge] = out_v
            new_sizes[lo:lo + cnt] = ns
            budget = math.ceil((1.0 + eps_l) * info.n_g / r)   # ams.py:258
            info.stats["over_budget"] = info.plan.max_load > budget
            infos.append(info)
            step = cnt // r
            next_groups.extend((lo + i * step, step) for i in range(r))
        buf, vbuf, obuf, sizes, groups = new_buf, new_vbuf, new_obuf, new_sizes, next_groups
        all_levels.append(infos)
        rep = {"level": lv + 1, "r": r, "max_load": max(sizes),
               "min_load": min(sizes),
               "sample_size": max(i.sample_size for i in infos),
               "plan_load": max(i.plan.max_load for i in infos),
               "over_budget": sum(bool(i.stats.get("over_budget")) for i in infos)}
        if with_stats:
            for key in ("max_words", "max_msgs", "max_sent_msgs", "max_recv_msgs"):
                rep[key] = max(i.stats[key] for i in infos)
        reports.append(rep)
    # Final local sort by (key, origin) (ams.py:310-312; a stable key sort
    # under "simple", F6).
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    for pe in range(p):
        s, e = int(offs[pe]), int(offs[pe + 1])
        order = np.lexsort((obuf[s:e], buf[s:e]))
        buf[s:e] = buf[s:e][order]
        if vbuf is not None:
            vbuf[s:e] = vbuf[s:e][order]
    return SortResult(buf, vbuf, sizes, all_levels, reports)


# --------------------------------------------------------------------------
# Inputs  (bench.py:153-177 for the reference generators)

def reference_uniform_input(p: int, n_per_pe: int, seed: int, rep: int = 0) -> np.ndarray:
    """The reference's ``generate_input(dist="uniform")`` keys
    (bench.py:159-164): PE stream ``input/rep{rep}/pe{pe}``,
    ``getrandbits(64)`` per key."""
    out = np.empty(p * n_per_pe, dtype=U64)
    for pe in range(p):
        rng = random.Random(stream_seed_int(seed, f"input/rep{rep}/pe{pe}"))
        # getrandbits(64 * n) packs n draws little-endian, identical to n
        # successive getrandbits(64) calls.
        big = rng.getrandbits(64 * n_per_pe) if n_per_pe else 0
        out[pe * n_per_pe:(pe + 1) * n_per_pe] = np.frombuffer(
            big.to_bytes(8 * n_per_pe, "little"), dtype="<u8")
    return out


_ZIPF_UNIVERSE = 100_000                                       # bench.py:137
_zipf_cache: dict = {}


def _zipf_cdf(theta: float) -> list:
    """bench.py:141-150 (same float accumulation order)."""
    cdf = _zipf_cache.get(theta)
    if cdf is None:
        acc = 0.0
        cdf = []
        for k in range(1, _ZIPF_UNIVERSE + 1):
            acc += k ** -theta
            cdf.append(acc)
        _zipf_cache[theta] = cdf
    return cdf


def reference_input(dist: str, p: int, n_per_pe: int, seed: int, rep: int = 0) -> np.ndarray:
    """All of ``generate_input``'s distributions (bench.py:153-177) as one
    PE-major uint64 array (origin tag of index i = (i // n_per_pe,
    i % n_per_pe))."""
    from bisect import bisect_left
    n = p * n_per_pe
    if dist == "uniform":
        return reference_uniform_input(p, n_per_pe, seed, rep)
    if dist == "sorted":
        return np.arange(n, dtype=U64)
    if dist == "reverse":
        return (n - 1 - np.arange(n, dtype=np.int64)).astype(U64)
    if dist == "equal":
        return np.full(n, 42, dtype=U64)
    if dist.startswith("zipf:"):
        theta = float(dist.split(":", 1)[1])
        cdf = _zipf_cdf(theta)
        total = cdf[-1]
        out = np.empty(n, dtype=U64)
        for pe in range(p):
            rng = random.Random(stream_seed_int(seed, f"input/rep{rep}/pe{pe}"))
            out[pe * n_per_pe:(pe + 1) * n_per_pe] = [
                bisect_left(cdf, rng.random() * total) for _ in range(n_per_pe)]
        return out
    raise ValueError(f"unknown input distribution {dist!r}")


def zipf_keys(n: int, seed: int, s: float = 1.1, universe: int = 1024) -> np.ndarray:
    """Config 4(a): Zipf(s) ranks 1..universe by inverse CDF."""
    rng = np.random.default_rng(seed)
    w = np.arange(1, universe + 1, dtype=np.float64) ** -s
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    u = rng.random(n)
    return (np.searchsorted(cdf, u, side="left") + 1).astype(U64)


def f64_to_ordered_u64(x: np.ndarray) -> np.ndarray:
    """Order-preserving float64 → uint64 map (sign-flip transform)."""
    b = np.ascontiguousarray(x, dtype=np.float64).view(U64)
    neg = (b >> U64(63)).astype(bool)
    return np.where(neg, ~b, b | U64(1 << 63))
