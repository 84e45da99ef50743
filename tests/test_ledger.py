"""Ledger parity: the reference's ``CostLedger`` state
after ``ams_sort(scheme="simple")`` replayed from per-level facts.

Fixtures: ``tests/golden/ledger/cases.json`` from the real reference
(``oracle/make_ledger_goldens.py``).  CPU tests feed the ledger replay with the
oracle's level facts; the GPU test feeds it with the device run's level records
through the drop-in ``api.ams_sort``.
"""

import json
import os

import numpy as np
import pytest

from paper_1410_6754_b200 import ledger as LG
from tests.simnet_standin import Costs, Net

CASES_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ledger",
                          "cases.json")


def cases():
    with open(CASES_PATH) as f:
        return json.load(f)


def case_keys(c):
    n = sum(c["sizes"])
    dist = c.get("dist", "uniform")
    if dist == "sorted":
        return np.arange(n, dtype=np.uint64)
    if dist == "reverse":
        return (n - 1 - np.arange(n)).astype(np.uint64)
    return np.random.default_rng(c["key_seed"]).integers(0, 2**64, n, dtype=np.uint64)


def ledger_state(ledger) -> dict:
    phases = {
        name: {"modeled_time": t.modeled_time, "sent_words": list(t.sent_words),
               "recv_words": list(t.recv_words), "sent_msgs": list(t.sent_msgs),
               "recv_msgs": list(t.recv_msgs), "coll_words": list(t.coll_words)}
        for name, t in ledger.phases.items()
    }
    return {"modeled_time": ledger.modeled_time, "sent_words": list(ledger.sent_words),
            "recv_words": list(ledger.recv_words), "sent_msgs": list(ledger.sent_msgs),
            "recv_msgs": list(ledger.recv_msgs), "coll_words": list(ledger.coll_words),
            "phases": phases, "phase_summary": ledger.phase_summary()}


def assert_ledger(ledger, ref):
    mine = ledger_state(ledger)
    assert list(mine["phases"]) == list(ref["phases"])      # phase order too
    for name in ref["phases"]:
        for k, v in ref["phases"][name].items():
            assert mine["phases"][name][k] == v, (name, k)
    for k in ("sent_words", "recv_words", "sent_msgs", "recv_msgs", "coll_words"):
        assert mine[k] == ref[k], k
    assert mine["modeled_time"] == ref["modeled_time"]       # bit-exact float
    assert mine["phase_summary"] == ref["phase_summary"]


@pytest.mark.parametrize("c", cases(), ids=lambda c: c["name"])
def test_ledger_from_oracle_levels(c):
    from oracle import ams_oracle as O

    keys = case_keys(c)
    res = O.ams_sort(keys, c["sizes"], tuple(c["groups"]), oversampling=c["a"],
                     overpartition=c["b"], imbalance=c["eps"], master_seed=c["master_seed"],
                     stream=c["stream"], scheme=c["scheme"])
    a = c["a"] if c["a"] is not None else O.default_oversampling(len(keys))
    net = Net(len(c["sizes"]), Costs(alpha=c["alpha"], beta=c["beta"]))
    for lv, infos in enumerate(res.levels):
        for info in infos:
            LG.charge_group_level(net, info.group_lo, info.hist, info.plan.boundaries,
                                  c["groups"][lv], c["b"], a, info.splitter_pos,
                                  scheme=c["scheme"], master_seed=c["master_seed"],
                                  level_stream=f"{c['stream']}/L{lv}-g{info.group_lo}")
    assert_ledger(net.ledger, c["ledger"])


def test_stand_in_ledger_semantics():
    net = Net(3, Costs(alpha=2.0, beta=0.5))
    with net.ledger.phase("x"):
        net.ledger.charge_collective([0, 1], 4, 3.0)
        net.ledger.record_exchange([2, 0, 0], [0, 0, 2], [1, 0, 0], [0, 0, 1], 3.0)
    with pytest.raises(RuntimeError):
        net.ledger.record_exchange([1, 0, 0], [0, 0, 0], [0, 0, 0], [0, 0, 0], 0.0)
    assert net.ledger.phase_summary()["x"] == {"modeled_time": 6.0, "max_words": 6,
                                               "max_msgs": 1}
    with pytest.raises(ValueError):
        Costs(alpha=-1.0)
    with pytest.raises(ValueError):
        Net(0)


def test_bucket_count_mismatch_rejected():
    hist = np.array([[3, 2], [1, 4]])
    net = Net(2)
    with pytest.raises(ValueError):
        LG.charge_group_level(net, 0, hist, [0, 1, 2], 2, 16, 10.0, [4])


@pytest.mark.gpu
@pytest.mark.parametrize("c", cases(), ids=lambda c: c["name"])
def test_ledger_through_dropin_api(c):
    """The drop-in ``ams_sort`` charges the caller's ledger like the reference."""
    from paper_1410_6754_b200 import api
    from paper_1410_6754_b200.params import AmsParams, Element, SeedSpec

    keys = case_keys(c)
    data, off = {}, 0
    for pe, s in enumerate(c["sizes"]):
        data[pe] = [Element(int(k), pe, i) for i, k in enumerate(keys[off:off + s])]
        off += s
    net = Net(len(c["sizes"]), Costs(alpha=c["alpha"], beta=c["beta"]))
    params = AmsParams(tuple(c["groups"]), oversampling=c["a"], overpartition=c["b"],
                       imbalance=c["eps"])
    out, reports = api.ams_sort(net, data, params, c["scheme"],
                                SeedSpec(c["master_seed"], c["stream"]))
    assert_ledger(net.ledger, c["ledger"])
    for mine, ref in zip(reports, c["reports"]):
        for k, v in ref.items():
            assert mine[k] == v, (k, mine[k], v)
    flat = sorted(int(k) for k in keys)
    assert [e.key for pe in range(len(c["sizes"])) for e in out[pe]] == flat


# --------------------------------------------------------------------------
# Whole experiment records (bench.py:180-242)

RECORDS_PATH = os.path.join(os.path.dirname(CASES_PATH), "records.jsonl")
PHASES = ("splitter_selection", "bucket_processing", "data_delivery", "local_sorting")


def records():
    with open(RECORDS_PATH) as f:
        return [line for line in f.read().splitlines() if line]


def experiment_record(ref: dict, a: float, pe_sizes, reports, net, verdict: str) -> str:
    """The record ``bench._run_once`` assembles (bench.py:207-242), from our
    sort's outputs and ledger; ``ref`` supplies the config fields."""
    pes, n_per_pe = ref["pes"], ref["n_per_pe"]
    avg = pes * n_per_pe / pes if pes else 0.0
    levels = [dict(r) for r in reports]
    for lv in levels:
        lv["imbalance"] = (lv["max_load"] / avg) if avg else 0.0
    phases = {name: {"modeled_time": 0.0, "max_words": 0, "max_msgs": 0} for name in PHASES}
    phases.update(net.ledger.phase_summary())
    loads = [int(x) for x in pe_sizes]
    rec = {k: ref[k] for k in ("schema", "algo", "pes", "n_per_pe", "levels", "groups")}
    rec["a"] = a
    rec.update({k: ref[k] for k in ("b", "eps", "delivery", "dist", "alpha", "beta", "seed",
                                    "rep")})
    rec.update({
        "verified": verdict,
        "final_max_load": max(loads),
        "final_imbalance": (max(loads) / avg) if avg else 0.0,
        "modeled_time": net.ledger.modeled_time,
        "max_sent_msgs": max(net.ledger.sent_msgs),
        "max_recv_msgs": max(net.ledger.recv_msgs),
        "phases": phases,
        "level_reports": levels,
    })
    return json.dumps(rec, separators=(",", ":"))


def record_input(ref):
    from oracle import ams_oracle as O
    return O.reference_input(ref["dist"], ref["pes"], ref["n_per_pe"], ref["seed"], ref["rep"])


@pytest.mark.parametrize("line", records(), ids=lambda s: "{delivery}-{dist}-{rep}".format(**json.loads(s)))
def test_record_from_oracle_levels(line):
    from oracle import ams_oracle as O

    ref = json.loads(line)
    keys = record_input(ref)
    groups = tuple(ref["groups"])
    res = O.ams_sort(keys, [ref["n_per_pe"]] * ref["pes"], groups, oversampling=ref["a"],
                     overpartition=ref["b"], imbalance=ref["eps"], master_seed=ref["seed"],
                     stream=f"algo/rep{ref['rep']}", scheme=ref["delivery"])
    net = Net(ref["pes"], Costs(alpha=ref["alpha"], beta=ref["beta"]))
    for lv, infos in enumerate(res.levels):
        for info in infos:
            LG.charge_group_level(net, info.group_lo, info.hist, info.plan.boundaries,
                                  groups[lv], ref["b"], ref["a"], info.splitter_pos,
                                  scheme=ref["delivery"], master_seed=ref["seed"],
                                  level_stream=f"algo/rep{ref['rep']}/L{lv}-g{info.group_lo}")
    verdict = "pass" if np.array_equal(res.keys, np.sort(keys)) else "fail"
    assert experiment_record(ref, ref["a"], res.pe_sizes, res.reports, net, verdict) == line


@pytest.mark.gpu
@pytest.mark.parametrize("line", records(), ids=lambda s: "{delivery}-{dist}-{rep}".format(**json.loads(s)))
def test_record_through_dropin_api(line):
    """``run_experiment``'s record, byte for byte, with the sort on the GPU."""
    from paper_1410_6754_b200 import api
    from paper_1410_6754_b200.params import AmsParams, Element, SeedSpec

    ref = json.loads(line)
    keys = record_input(ref)
    npe = ref["n_per_pe"]
    data = {pe: [Element(int(k), pe, i) for i, k in enumerate(keys[pe * npe:(pe + 1) * npe])]
            for pe in range(ref["pes"])}
    net = Net(ref["pes"], Costs(alpha=ref["alpha"], beta=ref["beta"]))
    params = AmsParams(tuple(ref["groups"]), oversampling=ref["a"], overpartition=ref["b"],
                       imbalance=ref["eps"])
    out, reports = api.ams_sort(net, data, params, ref["delivery"],
                                SeedSpec(ref["seed"], "algo").derive(f"rep{ref['rep']}"))
    flat = [e for pe in range(ref["pes"]) for e in out[pe]]
    expected = sorted(e for seq in data.values() for e in seq)
    verdict = "pass" if flat == expected else "fail"
    sizes = [len(out[pe]) for pe in range(ref["pes"])]
    assert experiment_record(ref, ref["a"], sizes, reports, net, verdict) == line
