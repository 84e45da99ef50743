"""Pin the CPU oracle to the real reference's outputs (golden fixtures).

The oracle (oracle/ams_oracle.py) is the checker for every GPU parity test;
these CPU tests show it reproduces the reference bit for bit: input
generation, sample streams, splitters, histograms, plans, per-PE sizes,
level reports, final output and origin permutation.
"""

import numpy as np
import pytest

from oracle import ams_oracle as O
from tests import golden_util as G

FAST = [n for n in G.names() if not n.startswith(("cfg1", "cfg2", "cfg3"))]
BIG = ["cfg1", "cfg2_scaled", "cfg3_scaled"]


def check_against_golden(g, res, keys):
    assert G.sha_u64(keys) == g["input_sha256"]
    assert list(res.pe_sizes) == g["pe_sizes"]
    assert G.sha_u64(res.keys) == g["output_sha256"]
    assert G.sha_i64(res.vals) == g["origin_sha256"]
    assert len(res.levels) == len(g["levels"])
    for lv, (mine, ref) in enumerate(zip(res.levels, g["levels"])):
        assert len(mine) == len(ref)
        for info, rg in zip(mine, ref):
            assert info.group_lo == rg["group_lo"]
            assert info.n_g == rg["n_g"]
            assert info.sample_size == rg["sample_size"]
            assert info.bucket_count == rg["bucket_count"]
            assert [int(x) for x in info.splitter_keys] == rg["splitter_keys"]
            assert [int(x) for x in info.splitter_pos] == rg["splitter_pos"]
            assert [int(x) for x in info.hist.sum(axis=0)] == rg["global_hist"]
            assert list(info.plan.boundaries) == rg["boundaries"]
            assert list(info.plan.loads) == rg["loads"]
            assert info.new_sizes == rg["new_sizes"]
    for mine, ref in zip(res.reports, g["reports"]):
        for k, v in ref.items():
            assert mine[k] == v, (k, mine[k], v)


def run_oracle(g):
    keys, sizes = G.input_of(g)
    vals = np.arange(len(keys), dtype=np.int64)
    res = O.ams_sort(keys, sizes, tuple(g["groups"]), g["a"], g["b"], g["eps"],
                     g["master_seed"], g["stream"], vals=vals, scheme=g.get("scheme", "simple"))
    return res, keys


@pytest.mark.parametrize("name", FAST)
def test_oracle_matches_reference_golden(name):
    g = G.load(name)
    if "error" in g:  # the reference rejects this input: same exception class and message
        exc = {"ValueError": ValueError, "RuntimeError": RuntimeError}[g["error"]["type"]]
        with pytest.raises(exc) as ei:
            run_oracle(g)
        assert str(ei.value) == g["error"]["message"]
        return
    res, keys = run_oracle(g)
    check_against_golden(g, res, keys)
    assert np.array_equal(res.keys, np.sort(keys))


@pytest.mark.parametrize("name", BIG)
def test_oracle_matches_reference_golden_big(name):
    g = G.load(name)
    res, keys = run_oracle(g)
    check_against_golden(g, res, keys)


def test_cfg1_survey_values():
    """SURVEY §8(c) recorded config-1 values."""
    g = G.load("cfg1")
    assert g["input_sha256"].startswith("63b56af9dbe0d121")
    assert g["levels"][0][0]["max_load"] == 66819
    keys, _ = G.input_of(g)
    assert int(keys[0]) == 0x2210358f89e992de


# Hand-traced plan cases (test_ams.py:29-63).
def test_plan_hand_cases():
    plan, _ = O._scan([5, 3, 4, 2, 6], 3, 8)
    assert plan.boundaries == (0, 2, 4, 5) and plan.loads == (8, 6, 6)
    assert O._scan([5, 3, 4, 2, 6], 3, 7)[0] is None
    assert O._scan([5, 3, 4], 3, 5)[0].loads == (5, 3, 4)
    assert O._scan([5, 3], 2, 4)[0] is None
    assert O.group_plan([5, 3, 4, 2, 6], 3).max_load == 8
    assert O.group_plan([5, 3, 4, 2, 6], 1).max_load == 20
    assert O.group_plan([5, 3, 4, 2, 6], 7).max_load == 6
    assert O.group_plan([0, 0, 0], 2).max_load == 0
