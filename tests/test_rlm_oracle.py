"""Pin the RLM-sort CPU oracle (oracle/rlm_oracle.py) to the real reference's
outputs: per-PE outputs, cut matrices (rlm.py:53-83), sizes, level reports."""

import numpy as np
import pytest

from oracle import rlm_oracle as R
from tests import rlm_golden_util as RG


def run(g):
    keys, sizes = RG.input_of(g)
    return keys, R.rlm_sort(keys, sizes, tuple(g["groups"]), g["scheme"], g["master_seed"], g["stream"])


@pytest.mark.parametrize("name", RG.NAMES)
def test_rlm_oracle_matches_reference_golden(name):
    g = RG.CASES[name]
    if "error" in g:
        exc = {"ValueError": ValueError, "RuntimeError": RuntimeError}[g["error"]["type"]]
        with pytest.raises(exc) as ei:
            run(g)
        assert str(ei.value) == g["error"]["message"]
        return
    keys, res = run(g)
    cuts = [[i.cuts for i in infos] for infos in res.levels]
    sizes_after = []
    for infos in res.levels:
        s = []
        for i in infos:
            s.extend(i.new_sizes)
        sizes_after.append(s)
    RG.check(g, keys, res.keys, res.origin, res.pe_sizes, cuts, sizes_after, res.reports)
    assert np.array_equal(res.keys, np.sort(keys))


def test_level_plan_validation():
    R.level_plan_check(16, (4, 4))
    for p, gc in ((16, (4, 2)), (16, (3, 4)), (0, (1,))):
        with pytest.raises(ValueError):
            R.level_plan_check(p, gc)
