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


# ---------------------------------------------------------------------------
# The full-size oracle (oracle/fullsize.py) used by the GPU tests at 2^28-2^30
# keys: same splitters, histograms, plans, member sizes and output as the
# pinned oracle and the reference's fixtures.

def _check_fullsize_against_golden(g):
    from oracle import fullsize as F
    keys, sizes = G.input_of(g)
    res = F.ams_sort_fullsize(keys, sizes, tuple(g["groups"]), g["a"], g["b"], g["eps"],
                              g["master_seed"], g["stream"], threads=4)
    assert list(res.pe_sizes) == g["pe_sizes"]
    assert G.sha_u64(res.keys) == g["output_sha256"]
    for facts, ref in zip(res.levels, g["levels"]):
        assert len(facts) == len(ref)
        for f, rg in zip(facts, ref):
            assert f.group_lo == rg["group_lo"] and f.n_g == rg["n_g"]
            assert f.sample_size == rg["sample_size"] and f.bucket_count == rg["bucket_count"]
            assert [int(x) for x in f.splitter_keys] == rg["splitter_keys"]
            assert [int(x) for x in f.hist.sum(axis=0)] == rg["global_hist"]
            assert list(f.boundaries) == rg["boundaries"] and list(f.loads) == rg["loads"]
            assert f.new_sizes == rg["new_sizes"]


SIMPLE_FAST = [n for n in FAST if G.load(n).get("scheme", "simple") == "simple"
               and "error" not in G.load(n)]


@pytest.mark.parametrize("name", SIMPLE_FAST + ["cfg2_scaled", "cfg3_scaled"])
def test_fullsize_oracle_matches_reference_golden(name):
    _check_fullsize_against_golden(G.load(name))


@pytest.mark.parametrize("groups,npe,dist", [
    ((8, 8), 700, "uniform"), ((8, 32), 90, "zipf"), ((4, 2, 2), 333, "equal"),
    ((16,), 1000, "sorted"), ((8, 4), 257, "reverse"), ((256,), 40, "uniform"),
])
def test_fullsize_matches_oracle(groups, npe, dist):
    """Per-level histograms, plans, member sizes and the final buffer equal
    ams_oracle.ams_sort's (ragged PE sizes too)."""
    from oracle import fullsize as F
    p = int(np.prod(groups))
    rng = np.random.default_rng(npe)
    sizes = [int(x) for x in rng.integers(npe // 2, 2 * npe, p)]
    n = sum(sizes)
    keys = {"uniform": lambda: rng.integers(0, 2**64, n, dtype=np.uint64),
            "zipf": lambda: O.zipf_keys(n, 7),
            "equal": lambda: np.full(n, 5, np.uint64),
            "sorted": lambda: np.arange(n, dtype=np.uint64),
            "reverse": lambda: (n - 1 - np.arange(n)).astype(np.uint64)}[dist]()
    ref = O.ams_sort(keys, sizes, groups, None, 16, 0.1, 3, "algo/rep0", with_stats=False)
    res = F.ams_sort_fullsize(keys, sizes, groups, None, 16, 0.1, 3, "algo/rep0", threads=3)
    assert np.array_equal(res.keys, ref.keys)
    assert list(res.pe_sizes) == list(ref.pe_sizes)
    for facts, infos in zip(res.levels, ref.levels):
        for f, info in zip(facts, infos):
            assert np.array_equal(f.hist, info.hist)
            assert tuple(f.boundaries) == tuple(info.plan.boundaries)
            assert f.new_sizes == list(info.new_sizes)
            assert np.array_equal(f.splitter_keys, info.splitter_keys)
