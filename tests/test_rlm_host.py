"""Host-side pieces of the RLM path (no GPU): LevelPlan validation
(rlm.py:22-45) and the deliver_simple planner of the C ABI against the
oracle's restatement (delivery.py:78-180)."""

import numpy as np
import pytest

from oracle import ams_oracle as O
from oracle import rlm_oracle as R


def test_level_plan_matches_reference_messages():
    from paper_1410_6754_b200.rlm import LevelPlan
    assert LevelPlan(16, (4, 4)).levels == 2
    for p, gc in ((16, (4, 2)), (16, (3, 4)), (0, (1,)), (8, (2, 0, 4))):
        with pytest.raises(ValueError) as e1:
            LevelPlan(p, gc)
        with pytest.raises(ValueError) as e2:
            R.level_plan_check(p, gc)
        assert str(e1.value) == str(e2.value)


@pytest.mark.parametrize("P,r", [(4, 2), (8, 8), (12, 3), (16, 4), (6, 1)])
def test_deliver_simple_matches_oracle(P, r):
    from paper_1410_6754_b200 import _lib as L
    rng = np.random.default_rng(P * 31 + r)
    for trial in range(20):
        pieces = rng.integers(0, 50, (P, r)).astype(np.uint64)
        if trial % 4 == 0:
            pieces[rng.integers(0, P)] = 0
        ns = np.zeros(P, np.uint64)
        st = np.zeros(4, np.uint64)
        L.check(L.lib.ams_deliver_simple(P, r, pieces.ctypes.data, ns.ctypes.data, st.ctypes.data))
        sub = P // r
        want = []
        for g in range(r):
            m = int(pieces[:, g].sum())
            want.extend((m * (t + 1)) // sub - (m * t) // sub for t in range(sub))
        assert [int(x) for x in ns] == want
        ref = O._exchange_stats(pieces.astype(np.int64), sub, list(range(P)))
        assert [int(x) for x in st] == [ref["max_words"], ref["max_msgs"], ref["max_sent_msgs"],
                                        ref["max_recv_msgs"]]
    with pytest.raises(ValueError):
        L.check(L.lib.ams_deliver_simple(5, 2, pieces.ctypes.data, ns.ctypes.data, None))
