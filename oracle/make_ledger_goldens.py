"""Ledger fixtures from the REAL reference — TEST INFRASTRUCTURE ONLY.

Runs ``mlpsort.ams.ams_sort`` (scheme ``"simple"``) from the read-only
``/root/reference`` on a fresh ``Network`` and records its ``CostLedger``
(simnet.py:139-256): per-PE totals, modeled time and every phase's tally.
The inputs are regenerated in the tests from the recorded seed
(``numpy.random.default_rng(seed).integers(0, 2**64)``, PE-major blocks), so
the fixtures hold only parameters and ledger state.

    python oracle/make_ledger_goldens.py      # writes tests/golden/ledger/cases.json
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import reference_loader  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "ledger", "cases.json")

# name, sizes per PE (or n_per_pe), group_counts, oversampling a, b, eps,
# key seed, master seed, alpha, beta
CASES = [
    ("flat16", 16, 1024, (16,), 16.0, 16, 0.1, 11, 0, 1.0, 1.0),
    ("two_level_64", 64, 512, (8, 8), None, 16, 0.1, 12, 1, 1.0, 1.0),
    ("two_level_8_frac", 8, 700, (2, 4), None, 8, 0.2, 13, 5, 0.37, 1.3),
    ("non_pow2_12", 12, 300, (3, 4), 4.0, 4, 0.2, 14, 7, 2.5, 0.75),
    ("three_level_16", 16, 256, (2, 2, 4), None, 16, 0.3, 15, 3, 1.0, 0.5),
    ("ragged_6", [0, 37, 5, 200, 1, 90], None, (2, 3), 2.0, 4, 0.2, 16, 9, 1.0, 1.0),
    ("single_pe", 1, 1000, (1,), None, 16, 0.1, 17, 2, 1.0, 1.0),
    # other delivery schemes (scheme, dist)
    ("det_two_level_64", 64, 512, (8, 8), None, 16, 0.1, 12, 1, 1.0, 1.0, "deterministic"),
    ("det_non_pow2_12", 12, 300, (3, 4), 4.0, 4, 0.2, 14, 7, 2.5, 0.75, "deterministic"),
    ("det_sorted_16", 16, 400, (4, 4), None, 8, 0.2, 18, 4, 0.3, 1.7, "deterministic", "sorted"),
    ("det_reverse_8", 8, 333, (8,), None, 16, 0.2, 19, 6, 1.0, 1.0, "deterministic", "reverse"),
    ("det_three_level_16", 16, 256, (2, 2, 4), None, 16, 0.3, 15, 3, 1.0, 0.5, "deterministic"),
    ("perm_two_level_64", 64, 512, (8, 8), None, 16, 0.1, 12, 1, 1.0, 1.0, "permuted"),
    ("perm_sorted_16", 16, 400, (4, 4), None, 8, 0.2, 18, 4, 0.3, 1.7, "permuted", "sorted"),
    ("rand_two_level_64", 64, 512, (8, 8), None, 16, 0.1, 12, 1, 1.0, 1.0, "randomized"),
    ("rand_sorted_16", 16, 400, (4, 4), None, 8, 0.2, 18, 4, 0.3, 1.7, "randomized", "sorted"),
    ("rand_reverse_32", 32, 200, (4, 8), None, 16, 0.2, 20, 8, 1.0, 1.0, "randomized",
     "reverse"),
    ("rand_flat_8", 8, 900, (8,), 3.0, 4, 0.2, 21, 10, 0.6, 1.1, "randomized", "sorted"),
    ("perm_ragged_6", [0, 37, 5, 200, 1, 90], None, (2, 3), 2.0, 4, 0.2, 16, 9, 1.0, 1.0,
     "permuted"),
]


OUT_RECORDS = os.path.join(ROOT, "tests", "golden", "ledger", "records.jsonl")
RECORD_CONFIGS = [
    dict(pes=16, n_per_pe=2048, levels=1, groups=(16,), seed=3, reps=2, dist="uniform"),
    dict(pes=64, n_per_pe=256, levels=2, groups=(8, 8), seed=4, dist="zipf:1.1",
         alpha=0.5, beta=2.0),
    dict(pes=16, n_per_pe=500, levels=2, groups=(4, 4), seed=5, dist="reverse", a=3.0, b=8,
         eps=0.3),
    dict(pes=8, n_per_pe=300, levels=1, groups=(8,), seed=6, dist="equal"),
    # the CLI / bench default delivery (bench.py:50)
    dict(pes=16, n_per_pe=1024, levels=2, groups=(4, 4), seed=7, dist="uniform",
         delivery="deterministic"),
    dict(pes=32, n_per_pe=256, levels=2, groups=(4, 8), seed=8, dist="sorted",
         delivery="deterministic"),
    dict(pes=16, n_per_pe=512, levels=2, groups=(4, 4), seed=9, dist="uniform",
         delivery="permuted"),
    dict(pes=16, n_per_pe=512, levels=2, groups=(4, 4), seed=10, dist="sorted",
         delivery="randomized"),
]


def case_sizes(spec, npe):
    if isinstance(spec, list):
        return list(spec)
    return [npe] * spec


def case_keys(sizes, seed, dist="uniform"):
    n = sum(sizes)
    if dist == "sorted":
        return np.arange(n, dtype=np.uint64)
    if dist == "reverse":
        return (n - 1 - np.arange(n)).astype(np.uint64)
    return np.random.default_rng(seed).integers(0, 2**64, n, dtype=np.uint64)


def ledger_state(ledger) -> dict:
    phases = {}
    for name, t in ledger.phases.items():
        phases[name] = {
            "modeled_time": t.modeled_time,
            "sent_words": list(t.sent_words), "recv_words": list(t.recv_words),
            "sent_msgs": list(t.sent_msgs), "recv_msgs": list(t.recv_msgs),
            "coll_words": list(t.coll_words),
        }
    return {
        "modeled_time": ledger.modeled_time,
        "sent_words": list(ledger.sent_words), "recv_words": list(ledger.recv_words),
        "sent_msgs": list(ledger.sent_msgs), "recv_msgs": list(ledger.recv_msgs),
        "coll_words": list(ledger.coll_words),
        "phases": phases,
        "phase_summary": ledger.phase_summary(),
    }


def main():
    reference_loader.load()
    from mlpsort.ams import AmsParams, ams_sort
    from mlpsort.core import Element, SeedSpec
    from mlpsort.simnet import CostParams, Network

    out = []
    for name, spec, npe, groups, a, b, eps, kseed, mseed, alpha, beta, *rest in CASES:
        scheme = rest[0] if rest else "simple"
        dist = rest[1] if len(rest) > 1 else "uniform"
        sizes = case_sizes(spec, npe)
        keys = case_keys(sizes, kseed, dist)
        data, off = {}, 0
        for pe, s in enumerate(sizes):
            data[pe] = [Element(int(k), pe, i) for i, k in enumerate(keys[off:off + s])]
            off += s
        net = Network(len(sizes), CostParams(alpha=alpha, beta=beta))
        params = AmsParams(groups, oversampling=a, overpartition=b, imbalance=eps)
        seed = SeedSpec(mseed, "algo").derive("rep0")
        _, reports = ams_sort(net, data, params, scheme, seed)
        out.append({
            "name": name, "sizes": sizes, "groups": list(groups), "a": a, "b": b,
            "eps": eps, "key_seed": kseed, "master_seed": mseed, "stream": "algo/rep0",
            "alpha": alpha, "beta": beta, "scheme": scheme, "dist": dist, "reports": reports,
            "ledger": ledger_state(net.ledger),
        })
        print(name, net.ledger.modeled_time)
    with open(OUT, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", OUT)

    # Whole experiment records (bench.py:180-242):
    # what ``run_experiment`` writes as JSONL, ledger phases included.
    from mlpsort.bench import ExperimentConfig, run_experiment
    recs = []
    for kw in RECORD_CONFIGS:
        cfg = ExperimentConfig(algo="ams", verify=True, **{"delivery": "simple", **kw})
        for rec in run_experiment(cfg):
            recs.append(json.dumps(rec, separators=(",", ":")))
    with open(OUT_RECORDS, "w") as f:
        f.write("\n".join(recs) + "\n")
    print("wrote", OUT_RECORDS, len(recs))


if __name__ == "__main__":
    main()
