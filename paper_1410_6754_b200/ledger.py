"""Communication ledger of the simulated machine, charged from the device run.

The reference prices every sort on a ``CostLedger`` (simnet.py:139-256):
collectives charge ``beta*words + alpha*ceil(log2 P)`` per call, the data
exchange records real per-PE word / message counts at ``h*beta + r*alpha``,
all under the phase labels of ams.py:222-250.  The B200 path never builds
messages, but every number the ledger needs is a function of facts the
device run already returns per level and group (``engine.LevelRecord``):
member sizes, the per-member bucket histogram, the plan boundaries and the
splitter positions.  :func:`charge_sort` replays the reference's charges
from those, in the reference's call order (so float sums match bit for bit),
onto the caller's ``net`` (the reference's ``mlpsort.simnet.Network`` or any
object with its ``.params.alpha/.beta`` and a ledger with ``phase``,
``record_exchange`` and ``charge_collective``; simnet.py:139-256).

Scope: the whole ``SCHEMES`` registry (delivery.py:138-455).
Host bookkeeping only; no device work happens here.
"""

from __future__ import annotations

import math

import numpy as np

PHASE_SPLITTERS = "splitter_selection"     # ams.py:222
PHASE_BUCKETS = "bucket_processing"        # ams.py:231
PHASE_DELIVERY = "data_delivery"           # ams.py:250


def _log2_ceil(n: int) -> int:
    """simnet.py:258-259."""
    return (n - 1).bit_length() if n > 1 else 0


# --------------------------------------------------------------------------
# Replaying the reference's charges

def _charge_vector(ledger, alpha, beta, members, length: int) -> None:
    """``Network.charge_vector_collective`` (simnet.py:367-371)."""
    n = len(members)
    if n > 1:
        ledger.charge_collective(members, length, length * beta + _log2_ceil(n) * alpha)


def _charge_gossip(ledger, alpha, beta, members, counts) -> None:
    """``Network.gossip_merge`` charge (simnet.py:373-396): every member
    receives the union minus its own contribution."""
    n = len(members)
    if n > 1:
        total = int(sum(counts))
        per = {pe: total - int(c) for pe, c in zip(members, counts)}
        ledger.charge_collective(members, per, max(per.values()) * beta + _log2_ceil(n) * alpha)


CHARGED_SCHEMES = ("simple", "deterministic", "permuted", "randomized")


def _mix64(x: int) -> int:
    """splitmix64 finalizer (core.py:74-79)."""
    x &= 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return x ^ (x >> 31)


def _feistel(n: int, seed):
    """``feistel_new(n, seed).apply`` (core.py:96-155): four keyed digit-pair
    rounds on the padded square domain, cycle-walked below n."""
    side = math.isqrt(n)
    if side * side < n:
        side += 1
    tables = [[_mix64(v ^ seed.key64(k)) % side for v in range(side)] for k in range(4)]

    def apply(i: int) -> int:
        x = i
        for _ in range(side * side):
            hi, lo = divmod(x, side)
            for t in tables:
                lo, hi = hi, (lo + t[hi]) % side
            x = lo + hi * side
            if x < n:
                return x
        raise RuntimeError("cycle walk failed to terminate")
    return apply


def _default_delegation_factor(p: int, r: int) -> int:
    """delivery.py:309-315."""
    if r * p <= 2:
        return 1
    a = 0.5 * (math.sqrt(1.0 + r / math.log(r * p / 2.0)) - 1.0)
    return max(1, math.floor(a))


def _charge_randomized(net, lo: int, pieces: np.ndarray, r: int, master_seed: int,
                       level_stream: str) -> None:
    """deliver_randomized's charges (delivery.py:318-436): delegation
    exchange, enumeration prefix sum, reply exchange, data exchange."""
    from .params import SeedSpec

    P = pieces.shape[0]
    members = list(range(lo, lo + P))
    sub = P // r
    seed = SeedSpec(master_seed, f"{level_stream}/deliver")
    n = int(pieces.sum())
    s = max(1, math.ceil(_default_delegation_factor(P, r) * n / (r * P)))
    chunks = []                                      # (idx, g, length, large)
    for idx in range(P):
        for g in range(r):
            size = int(pieces[idx, g])
            if size == 0:
                continue
            if size > s:
                whole, rem = divmod(size, s)
                chunks.extend((idx, g, s, True) for _ in range(whole))
                if rem:
                    chunks.append((idx, g, rem, False))
            else:
                chunks.append((idx, g, size, False))
    large_ids = [i for i, ch in enumerate(chunks) if ch[3]]
    holder_of = {}
    if large_ids:
        perm = _feistel(len(large_ids), seed.derive("delegate"))
        for rank, cid in enumerate(large_ids):
            holder_of[cid] = perm(rank) % P
    words: dict = {}                                 # (g, idx, offset, length) each
    for cid in large_ids:
        key = (chunks[cid][0], holder_of[cid])
        words[key] = words.get(key, 0) + 4
    _exchange(net, lo, P, [(a, b, w) for (a, b), w in words.items()])
    held: dict = {}
    for cid, (idx, g, _, _) in enumerate(chunks):
        held.setdefault((g, holder_of.get(cid, idx)), []).append(cid)
    start_of, totals = {}, [0] * r
    for g in range(r):
        order = _feistel(P, seed.derive(f"order-g{g}"))
        running = 0
        for holder in sorted(range(P), key=order):
            mine = held.get((g, holder), [])
            if not mine:
                continue
            seed.derive(f"reorder-g{g}-h{holder}").rng().shuffle(mine)
            for cid in mine:
                start_of[cid] = running
                running += chunks[cid][2]
        totals[g] = running
    _charge_vector(net.ledger, net.params.alpha, net.params.beta, members, r)
    words = {}                                       # (g, offset, start) each
    for cid in large_ids:
        idx, holder = chunks[cid][0], holder_of[cid]
        if holder != idx:
            words[(holder, idx)] = words.get((holder, idx), 0) + 3
    _exchange(net, lo, P, [(a, b, w) for (a, b), w in words.items()])
    msgs = []
    for cid, (idx, g, length, _) in enumerate(chunks):
        m, st = totals[g], start_of[cid]
        for t in range(sub):                         # quota slots (delivery.py:78-104)
            take = min(st + length, (m * (t + 1)) // sub) - max(st, (m * t) // sub)
            if take > 0:
                msgs.append((idx, g * sub + t, take))
    _exchange(net, lo, P, msgs)


def _exchange(net, lo: int, P: int, msgs) -> None:
    """``Network.exchange`` accounting (simnet.py:294-335) of one group's
    messages ``(src member, dest member, words)``; self-messages are free."""
    p_all = net.p
    sw, rw = [0] * p_all, [0] * p_all
    sm, rm = [0] * p_all, [0] * p_all
    for s, d, w in msgs:
        if w == 0 or s == d:
            continue
        sw[lo + s] += w
        rw[lo + d] += w
        sm[lo + s] += 1
        rm[lo + d] += 1
    members = range(lo, lo + P)
    h = max(max(sw[pe] for pe in members), max(rw[pe] for pe in members))
    m = max(max(sm[pe] for pe in members), max(rm[pe] for pe in members))
    net.ledger.record_exchange(sw, rw, sm, rm, h * net.params.beta + m * net.params.alpha)


def _simple_messages(pieces: np.ndarray, r: int):
    """deliver_simple's slices (delivery.py:78-104, 151-180): piece (j, g) at
    numbers [start, start+size) of subgroup g, cut along the quota slots."""
    P = pieces.shape[0]
    sub = P // r
    starts = np.cumsum(pieces, axis=0) - pieces                      # source order
    totals = pieces.sum(axis=0)
    t = np.arange(sub + 1, dtype=np.int64)
    msgs = []
    for g in range(r):
        cut = (int(totals[g]) * t) // sub
        s0 = starts[:, g][:, None]
        s1 = (starts[:, g] + pieces[:, g])[:, None]
        take = np.minimum(s1, cut[None, 1:]) - np.maximum(s0, cut[None, :-1])
        for j, d in zip(*np.nonzero(take > 0)):
            msgs.append((int(j), g * sub + int(d), int(take[j, d])))
    return msgs


def _planned_messages(pieces: np.ndarray, r: int, slices: np.ndarray, new_sizes):
    """Messages of a planner's slices (src offset in the group's simple
    layout, dst offset in the new member arrays, length), each tagged with its
    piece (j, g): [(src member, dest member, words, j, g)]."""
    P = pieces.shape[0]
    order = [(g, j) for g in range(r) for j in range(P)]             # (g, j, b) layout
    flat = np.array([pieces[j, g] for g, j in order], dtype=np.int64)
    pstart = np.concatenate([[0], np.cumsum(flat)])[:-1]
    nz = np.nonzero(flat)[0]
    noff = np.concatenate([[0], np.cumsum(np.asarray(new_sizes, dtype=np.int64))])
    out = []
    for src, dst, ln in np.asarray(slices, dtype=np.int64).reshape(-1, 3):
        k = nz[np.searchsorted(pstart[nz], src, side="right") - 1]
        g, j = order[k]
        d = int(np.searchsorted(noff, dst, side="right") - 1)
        out.append((j, d, int(ln), j, g))
    return out


def _charge_delivery(net, lo: int, pieces: np.ndarray, r: int, scheme: str,
                     master_seed, level_stream) -> None:
    ledger, alpha = net.ledger, net.params.alpha
    P = pieces.shape[0]
    members = list(range(lo, lo + P))
    if scheme == "simple":                                           # delivery.py:151-180
        _charge_vector(ledger, alpha, net.params.beta, members, r)
        _exchange(net, lo, P, _simple_messages(pieces, r))
        return
    from . import _lib as L
    if scheme == "permuted":                                         # delivery.py:183-185
        new_sizes, slices, _ = L.deliver_permuted(pieces, master_seed, level_stream, False)
        _charge_vector(ledger, alpha, net.params.beta, members, r)
        _exchange(net, lo, P, [m[:3] for m in _planned_messages(pieces, r, slices, new_sizes)])
        return
    if scheme == "randomized":
        _charge_randomized(net, lo, pieces, r, master_seed, level_stream)
        return
    if scheme != "deterministic":
        raise ValueError(f"ledger charges of scheme {scheme!r} are not modelled")
    # deliver_deterministic (delivery.py:188-306)
    new_sizes, slices, _ = L.deliver_deterministic(pieces, lo, False)
    msgs = _planned_messages(pieces, r, slices, new_sizes)
    n = int(pieces.sum())
    sub = P // r
    _charge_vector(ledger, alpha, net.params.beta, members, 2 * r)
    large = [(j, g) for g in range(r) for j in range(P)
             if pieces[j, g] > 0 and not int(pieces[j, g]) * 2 * P * r <= n]
    # descriptors (g, idx, size) to coordinator sub[idx // r], bundled per edge
    desc: dict = {}
    for j, g in large:
        key = (j, g * sub + j // r)
        desc[key] = desc.get(key, 0) + 3
    _exchange(net, lo, P, [(s, d, w) for (s, d), w in sorted(desc.items())])
    if sub > 1:                                                      # group-local merge
        ledger.charge_collective(members, 0, alpha * _log2_ceil(sub))
    # replies (g, dest, offset, length) per cut, coordinator -> origin, bundled
    cuts: dict = {}
    for _, _, _, j, g in msgs:
        cuts[(j, g)] = cuts.get((j, g), 0) + 1
    rep: dict = {}
    for j, g in large:
        key = (g * sub + j // r, j)
        rep[key] = rep.get(key, 0) + 4 * cuts[(j, g)]
    _exchange(net, lo, P, [(s, d, w) for (s, d), w in sorted(rep.items())])
    _exchange(net, lo, P, [m[:3] for m in msgs])


def charge_group_level(net, lo: int, hist: np.ndarray, boundaries, r: int, b: int, a: float,
                       splitter_pos=None, holders=None, scheme: str = "simple",
                       master_seed: int | None = None, level_stream: str | None = None) -> None:
    """Charges of one ``ams_level`` call (ams.py:214-268) on the group of PEs
    ``lo .. lo+P-1``.

    hist:         (P, br) per-member bucket histogram (row sums = member sizes)
    boundaries:   plan boundaries (r+1)
    splitter_pos: position in the group buffer of each splitter (br-1), or
    holders:      per member, how many splitters were drawn from it
    level_stream: "{stream}/L{level}-g{lo}" (the seeded schemes' Feistel orders)
    """
    ledger, alpha, beta = net.ledger, net.params.alpha, net.params.beta
    hist = np.asarray(hist, dtype=np.int64)
    P, br = hist.shape
    members = list(range(lo, lo + P))
    sizes = hist.sum(axis=1)
    n_g = int(sizes.sum())

    with ledger.phase(PHASE_SPLITTERS):
        # draw_sample quotas (ams.py:157-175, 224-228)
        br0 = min(b * r, n_g + 1)
        target = min(n_g, max(br0 - 1, math.ceil(a * br0)))
        base, extra = divmod(target, P)
        takes = np.minimum(base + (np.arange(P) < extra), sizes)
        drawn = int(takes.sum())
        if min(br0, drawn + 1) != br:
            raise ValueError(f"bucket count {br} does not match the sample of {drawn}")
        if br > 1:                                                   # ams.py:188-198
            wanted = sorted({(i * drawn) // br for i in range(1, br)})
            if P & (P - 1) == 0:
                # fast_rank_sort (fastsort.py:57-108): row and column gossips,
                # then one allreduce of the partial ranks per column.
                exp = P.bit_length() - 1
                rows, cols = 1 << ((exp + 1) // 2), 1 << (exp // 2)
                for i in range(rows):
                    idx = list(range(i * cols, (i + 1) * cols))
                    _charge_gossip(ledger, alpha, beta, [members[j] for j in idx], takes[idx])
                for j in range(cols):
                    idx = list(range(j, P, cols))
                    _charge_gossip(ledger, alpha, beta, [members[i] for i in idx], takes[idx])
                for j in range(cols):
                    idx = list(range(j, P, cols))
                    _charge_vector(ledger, alpha, beta, [members[i] for i in idx],
                                   int(takes[idx].sum()))
                # extract_by_ranks (fastsort.py:111-130): the holders of the
                # wanted ranks gossip them to every member.
                if holders is None:
                    pos = np.asarray(splitter_pos, dtype=np.int64)
                    offs = np.concatenate([[0], np.cumsum(sizes)])
                    holders = np.bincount(np.searchsorted(offs, pos, side="right") - 1,
                                          minlength=P)[:P]
                holders = np.asarray(holders, dtype=np.int64)
                if len(holders) != P or int(holders.sum()) != len(wanted):
                    raise ValueError("one splitter holder per wanted rank expected")
                _charge_gossip(ledger, alpha, beta, members, holders)
            else:                                                    # ams.py:195-197
                ledger.charge_collective(
                    members, drawn, 2 * (drawn * beta + _log2_ceil(P) * alpha))

    with ledger.phase(PHASE_BUCKETS):                                # ams.py:236-237
        _charge_vector(ledger, alpha, beta, members, br)

    with ledger.phase(PHASE_DELIVERY):
        bnd = np.asarray(boundaries, dtype=np.int64)
        pieces = np.stack([hist[:, bnd[g]:bnd[g + 1]].sum(axis=1) for g in range(r)], axis=1)
        _charge_delivery(net, lo, pieces, r, scheme, master_seed, level_stream)


def charge_sort(net, levels, params, a: float, scheme: str = "simple",
                master_seed: int | None = None, stream_id: str | None = None) -> None:
    """Every level's charges (ams.py:284-290), group by group in PE order, from
    the device run's level records (splitter holders or recorded splitters)."""
    if scheme not in CHARGED_SCHEMES:
        raise ValueError(f"ledger charges of scheme {scheme!r} are not modelled")
    b = params.overpartition
    for rec in levels:
        if rec.holders is None and not rec.splitters:
            raise ValueError("ledger charging needs each level's splitter holders")
        for gi in range(len(rec.group_first)):
            lo, P = int(rec.group_first[gi]), int(rec.group_npe[gi])
            br = int(rec.bucket_count[gi])
            hist = np.asarray(rec.seg_hist[lo:lo + P, :br], dtype=np.int64)
            if rec.holders is not None:
                kw = {"holders": np.asarray(rec.holders[lo:lo + P], dtype=np.int64)}
            else:
                _, pos = rec.splitters[gi]
                kw = {"splitter_pos": np.asarray(pos, dtype=np.int64)[:max(br - 1, 0)]}
            charge_group_level(net, lo, hist, rec.boundaries[gi], rec.r, b, a, scheme=scheme,
                               master_seed=master_seed,
                               level_stream=f"{stream_id}/L{rec.level}-g{lo}", **kw)
