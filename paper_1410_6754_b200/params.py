"""Parameter and record types of the AMS-sort entry point, restated with the
reference's names, fields and validation so callers can switch over
unchanged.

* ``AmsParams`` — ams.py:33-65 (same fields, defaults, errors).
* ``GroupPlan`` — ams.py:68-75.
* ``SeedSpec``  — core.py:46-71 (named replayable streams).
* ``Element``   — core.py:19-29 (key + origin tag).
"""

from __future__ import annotations

import hashlib
import math
import random
from dataclasses import dataclass
from typing import NamedTuple


class Element(NamedTuple):
    """One record: 64-bit key plus origin tag (core.py:19-29)."""

    key: int
    origin_pe: int
    origin_pos: int


@dataclass(frozen=True)
class AmsParams:
    """Per-level group counts (product = p), oversampling a, overpartitioning
    b, total imbalance eps (ams.py:33-65)."""

    group_counts: tuple
    oversampling: float | None = None
    overpartition: int = 16
    imbalance: float = 0.2

    def __post_init__(self):
        if not self.group_counts or any(r < 1 for r in self.group_counts):
            raise ValueError("group counts must be positive")
        if self.overpartition < 1:
            raise ValueError("overpartitioning factor must be at least 1")
        if self.oversampling is not None and self.oversampling <= 0:
            raise ValueError("oversampling factor must be positive")
        if self.imbalance <= 0:
            raise ValueError("imbalance budget must be positive")

    @property
    def levels(self) -> int:
        return len(self.group_counts)

    def per_level_imbalance(self) -> float:
        return (1.0 + self.imbalance) ** (1.0 / self.levels) - 1.0

    def validate_for(self, p: int) -> None:
        prod = math.prod(self.group_counts)
        if prod != p:
            raise ValueError(
                f"group counts {tuple(self.group_counts)} do not telescope {p} PEs")

    def oversampling_for(self, n: int) -> float:
        """ams.py:278-280."""
        a = self.oversampling
        return a if a is not None else 1.6 * math.log10(max(n, 10))


@dataclass(frozen=True)
class GroupPlan:
    """Consecutive bucket ranges per group (ams.py:68-75)."""

    boundaries: tuple
    loads: tuple
    max_load: int


@dataclass(frozen=True)
class SeedSpec:
    """Named, replayable random stream (core.py:46-71)."""

    master_seed: int
    stream_id: str = "root"

    def derive(self, label: str) -> "SeedSpec":
        return SeedSpec(self.master_seed, f"{self.stream_id}/{label}")

    def _digest(self, extra: str = "") -> bytes:
        text = f"{self.master_seed}\x1f{self.stream_id}\x1f{extra}"
        return hashlib.blake2b(text.encode(), digest_size=16).digest()

    def rng(self) -> random.Random:
        return random.Random(int.from_bytes(self._digest(), "big"))

    def key64(self, index: int) -> int:
        return int.from_bytes(self._digest(f"k{index}")[:8], "big")


def as_seed(seed) -> tuple[int, str]:
    """(master_seed, stream_id) of our SeedSpec or the reference's.  The seed
    crosses the C ABI as int64 and is hashed there as its decimal text
    (core.py:52-55 hashes f"{master_seed}"), so it must fit in int64."""
    m = int(seed.master_seed)
    if not -(1 << 63) <= m < (1 << 63):
        raise ValueError(f"master_seed {m} outside the supported int64 range")
    return m, str(seed.stream_id)


def as_params(params) -> AmsParams:
    """Accept the reference's AmsParams too (same fields)."""
    if isinstance(params, AmsParams):
        return params
    return AmsParams(tuple(params.group_counts), params.oversampling, params.overpartition,
                     params.imbalance)
