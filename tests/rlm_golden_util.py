"""RLM-sort golden fixtures (made by ``oracle/make_rlm_goldens.py`` from the
real reference) and the checks shared by the CPU-oracle and GPU tests."""

import json
import os

import numpy as np

from tests import golden_util as G

PATH = os.path.join(G.GOLDEN_DIR, "rlm", "cases.json")
with open(PATH) as _f:
    CASES = {c["name"]: c for c in json.load(_f)}
NAMES = sorted(CASES)


def input_of(g):
    from oracle import ams_oracle as O
    if "data" in g:
        keys = [k for pe in range(g["p"]) for k in g["data"][str(pe)]]
        return np.asarray(keys, dtype=np.uint64), list(g["input_pe_sizes"])
    return O.reference_input(g["dist"], g["p"], g["n_per_pe"], g["input_seed"]), list(g["input_pe_sizes"])


def check(g, keys, out_keys, out_origin, pe_sizes, level_cuts, level_sizes, reports):
    """level_cuts[lv][gi] = (P, r+1) cut matrix; level_sizes[lv] = member
    sizes after the level (all PEs); reports = list of dicts."""
    assert G.sha_u64(keys) == g["input_sha256"]
    assert [int(x) for x in pe_sizes] == g["pe_sizes"]
    assert G.sha_u64(out_keys) == g["output_sha256"]
    assert G.sha_i64(out_origin) == g["origin_sha256"]
    if "output" in g:
        assert [[int(k), int(o)] for k, o in zip(out_keys, out_origin)] == g["output"]
    assert len(level_cuts) == len(g["levels"])
    for mine, ref in zip(level_cuts, g["levels"]):
        assert len(mine) == len(ref)
        for cuts, rg in zip(mine, ref):
            assert [[int(x) for x in row] for row in np.asarray(cuts)] == rg["cuts"]
    for lv, ref in enumerate(g["reports"]):
        sizes = [int(x) for x in level_sizes[lv]]
        assert max(sizes) == ref["max_load"] and min(sizes) == ref["min_load"]
        for k, v in ref.items():
            assert int(reports[lv][k]) == v, (lv, k, reports[lv][k], v)
