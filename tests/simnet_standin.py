"""Test-only stand-in for the caller's ``mlpsort.simnet.Network`` (``.p`` and
``.ledger``): the ledger parity tests charge it through
``paper_1410_6754_b200.ledger.charge_sort`` and compare its counters with
the reference's fixtures.  The product never constructs one — the drop-in
``api.ams_sort`` charges whatever ``net`` the caller passes (duck-typed on
``phase`` / ``record_exchange`` / ``charge_collective``, the interface of
simnet.py:139-256).
"""

from __future__ import annotations

from contextlib import contextmanager

_FIELDS = ("sent_words", "recv_words", "sent_msgs", "recv_msgs", "coll_words")


class Costs:
    """alpha (message startup) and beta (per word); both non-negative."""

    def __init__(self, alpha: float = 1.0, beta: float = 1.0):
        if min(alpha, beta) < 0:
            raise ValueError("cost parameters must be non-negative")
        self.alpha, self.beta = alpha, beta


class Counters:
    """Per-PE word/message vectors plus the modelled time."""

    def __init__(self, p: int):
        self.modeled_time = 0.0
        for f in _FIELDS:
            setattr(self, f, [0] * p)


class Ledger(Counters):
    """Totals plus one :class:`Counters` per phase label, in first-use order."""

    def __init__(self, p: int, costs: Costs):
        super().__init__(p)
        self.p, self.params = p, costs
        self.phases: dict[str, Counters] = {}
        self._label = "setup"

    @contextmanager
    def phase(self, label: str):
        saved, self._label = self._label, label
        try:
            yield self
        finally:
            self._label = saved

    def _current(self) -> Counters:
        return self.phases.setdefault(self._label, Counters(self.p))

    def _add(self, field: str, pe: int, v: int, cur: Counters) -> None:
        getattr(self, field)[pe] += v
        getattr(cur, field)[pe] += v

    def record_exchange(self, sw, rw, sm, rm, cost: float) -> None:
        if sum(sw) != sum(rw) or sum(sm) != sum(rm):
            raise RuntimeError("exchange lost or duplicated traffic")
        cur = self._current()
        for pe, vals in enumerate(zip(sw, rw, sm, rm)):
            if any(vals):
                for field, v in zip(_FIELDS[:4], vals):
                    self._add(field, pe, v, cur)
        self.modeled_time += cost
        cur.modeled_time += cost

    def charge_collective(self, members, words, time: float) -> None:
        cur = self._current()
        per = words if isinstance(words, dict) else {pe: words for pe in members}
        for pe, w in per.items():
            self._add("coll_words", pe, w, cur)
        self.modeled_time += time
        cur.modeled_time += time

    def phase_summary(self) -> dict:
        return {
            label: {
                "modeled_time": c.modeled_time,
                "max_words": max((max(a, b) + w for a, b, w in
                                  zip(c.sent_words, c.recv_words, c.coll_words)), default=0),
                "max_msgs": max((max(a, b) for a, b in zip(c.sent_msgs, c.recv_msgs)),
                                default=0),
            }
            for label, c in self.phases.items()
        }


class Net:
    """``p`` PEs and their ledger."""

    def __init__(self, p: int, costs: Costs | None = None):
        if p < 1:
            raise ValueError("need at least one PE")
        self.p = p
        self.params = costs or Costs()
        self.ledger = Ledger(p, self.params)
