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
onto any object with the reference ledger's methods — the user's own
``mlpsort.simnet.Network``, or the stand-in :class:`Network` below.

Scope: ``scheme="simple"`` (delivery.py:138-180).  Host bookkeeping only; no
device work happens here.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

PHASE_SPLITTERS = "splitter_selection"     # ams.py:222
PHASE_BUCKETS = "bucket_processing"        # ams.py:231
PHASE_DELIVERY = "data_delivery"           # ams.py:250


def _log2_ceil(n: int) -> int:
    """simnet.py:258-259."""
    return (n - 1).bit_length() if n > 1 else 0


# --------------------------------------------------------------------------
# Stand-ins with the reference's interface (simnet.py:42-50, 123-256, 262-290)

@dataclass(frozen=True)
class CostParams:
    """Message startup cost (alpha) and per-word cost (beta); simnet.py:42-50."""

    alpha: float = 1.0
    beta: float = 1.0

    def __post_init__(self):
        if self.alpha < 0 or self.beta < 0:
            raise ValueError("cost parameters must be non-negative")


class _PhaseTally:
    __slots__ = ("modeled_time", "sent_words", "recv_words", "sent_msgs",
                 "recv_msgs", "coll_words")

    def __init__(self, p: int):
        self.modeled_time = 0.0
        self.sent_words = [0] * p
        self.recv_words = [0] * p
        self.sent_msgs = [0] * p
        self.recv_msgs = [0] * p
        self.coll_words = [0] * p


class CostLedger:
    """Per-PE exchange / collective counters with phase breakdown, same
    methods and semantics as the reference's (simnet.py:139-256)."""

    def __init__(self, p: int, params: CostParams):
        self.p = p
        self.params = params
        self.modeled_time = 0.0
        self.sent_words = [0] * p
        self.recv_words = [0] * p
        self.sent_msgs = [0] * p
        self.recv_msgs = [0] * p
        self.coll_words = [0] * p
        self._phase = "setup"
        self.phases: dict[str, _PhaseTally] = {}

    class _Scope:
        def __init__(self, ledger, name):
            self.ledger, self.name = ledger, name

        def __enter__(self):
            self.prev, self.ledger._phase = self.ledger._phase, self.name
            return self.ledger

        def __exit__(self, *exc):
            self.ledger._phase = self.prev
            return False

    def phase(self, name: str):
        return CostLedger._Scope(self, name)

    def _tally(self) -> _PhaseTally:
        t = self.phases.get(self._phase)
        if t is None:
            t = self.phases[self._phase] = _PhaseTally(self.p)
        return t

    def record_exchange(self, sw, rw, sm, rm, cost: float) -> None:
        if sum(sw) != sum(rw) or sum(sm) != sum(rm):
            raise RuntimeError("exchange lost or duplicated traffic")
        t = self._tally()
        for pe in range(self.p):
            if sw[pe] or rw[pe] or sm[pe] or rm[pe]:
                for name, vec in (("sent_words", sw), ("recv_words", rw),
                                  ("sent_msgs", sm), ("recv_msgs", rm)):
                    getattr(self, name)[pe] += vec[pe]
                    getattr(t, name)[pe] += vec[pe]
        self.modeled_time += cost
        t.modeled_time += cost

    def charge_collective(self, members, words_per_member, time: float) -> None:
        t = self._tally()
        per = ({pe: words_per_member for pe in members}
               if isinstance(words_per_member, int) else words_per_member)
        for pe, w in per.items():
            self.coll_words[pe] += w
            t.coll_words[pe] += w
        self.modeled_time += time
        t.modeled_time += time

    def phase_summary(self) -> dict:
        out = {}
        for name, t in self.phases.items():
            out[name] = {
                "modeled_time": t.modeled_time,
                "max_words": max((max(t.sent_words[pe], t.recv_words[pe]) + t.coll_words[pe]
                                  for pe in range(self.p)), default=0),
                "max_msgs": max((max(t.sent_msgs[pe], t.recv_msgs[pe])
                                 for pe in range(self.p)), default=0),
            }
        return out


class Network:
    """``p`` PEs plus their ledger (simnet.py:262-273), for callers without
    the reference package."""

    def __init__(self, p: int, params: CostParams | None = None):
        if p < 1:
            raise ValueError("need at least one PE")
        self.p = p
        self.params = params or CostParams()
        self.ledger = CostLedger(p, self.params)


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


def charge_group_level(net, lo: int, hist: np.ndarray, boundaries, r: int, b: int, a: float,
                       splitter_pos) -> None:
    """Charges of one ``ams_level`` call (ams.py:214-268) on the group of PEs
    ``lo .. lo+P-1`` with scheme "simple".

    hist:        (P, br) per-member bucket histogram (row sums = member sizes)
    boundaries:  plan boundaries (r+1)
    splitter_pos: position in the group buffer of each splitter (br-1)
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
                pos = np.asarray(splitter_pos, dtype=np.int64)
                if len(pos) != len(wanted):
                    raise ValueError("one splitter position per wanted rank expected")
                offs = np.concatenate([[0], np.cumsum(sizes)])
                holder = np.searchsorted(offs, pos, side="right") - 1
                contrib = np.bincount(holder, minlength=P)[:P]
                _charge_gossip(ledger, alpha, beta, members, contrib)
            else:                                                    # ams.py:195-197
                ledger.charge_collective(
                    members, drawn, 2 * (drawn * beta + _log2_ceil(P) * alpha))

    with ledger.phase(PHASE_BUCKETS):                                # ams.py:236-237
        _charge_vector(ledger, alpha, beta, members, br)

    with ledger.phase(PHASE_DELIVERY):                               # delivery.py:138-180
        _charge_vector(ledger, alpha, beta, members, r)
        bnd = np.asarray(boundaries, dtype=np.int64)
        pieces = np.stack([hist[:, bnd[g]:bnd[g + 1]].sum(axis=1) for g in range(r)], axis=1)
        starts = np.cumsum(pieces, axis=0) - pieces                  # source order
        totals = pieces.sum(axis=0)
        sub = P // r
        p_all = net.p
        sw, rw = [0] * p_all, [0] * p_all
        sm, rm = [0] * p_all, [0] * p_all
        t = np.arange(sub + 1, dtype=np.int64)
        src = np.arange(P)
        for g in range(r):
            cut = (int(totals[g]) * t) // sub                        # quota slots
            s0 = starts[:, g][:, None]
            s1 = (starts[:, g] + pieces[:, g])[:, None]
            take = np.minimum(s1, cut[None, 1:]) - np.maximum(s0, cut[None, :-1])
            take = np.where(take > 0, take, 0)
            dest = g * sub + np.arange(sub)
            take[src[:, None] == dest[None, :]] = 0                  # self-messages are free
            for j, d in zip(*np.nonzero(take)):
                w = int(take[j, d])
                s_pe, d_pe = lo + int(j), lo + int(dest[d])
                sw[s_pe] += w
                rw[d_pe] += w
                sm[s_pe] += 1
                rm[d_pe] += 1
        h = max(max(sw[pe] for pe in members), max(rw[pe] for pe in members))
        m = max(max(sm[pe] for pe in members), max(rm[pe] for pe in members))
        ledger.record_exchange(sw, rw, sm, rm, h * beta + m * alpha)  # simnet.py:294-335


def charge_sort(net, levels, params, a: float) -> None:
    """Every level's charges (ams.py:284-290), group by group in PE order, from
    the device run's level records (recorded splitters required)."""
    b = params.overpartition
    for rec in levels:
        if not rec.splitters:
            raise ValueError("ledger charging needs the recorded splitters of every level")
        for gi in range(len(rec.group_first)):
            lo, P = int(rec.group_first[gi]), int(rec.group_npe[gi])
            br = int(rec.bucket_count[gi])
            hist = np.asarray(rec.seg_hist[lo:lo + P, :br], dtype=np.int64)
            _, pos = rec.splitters[gi]
            charge_group_level(net, lo, hist, rec.boundaries[gi], rec.r, b, a,
                               np.asarray(pos, dtype=np.int64)[:max(br - 1, 0)])
