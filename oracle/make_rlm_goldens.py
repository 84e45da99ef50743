"""Generate RLM-sort golden fixtures from the REAL reference — TEST
INFRASTRUCTURE ONLY (run in the build container, where /root/reference exists):

    python -m oracle.make_rlm_goldens

Writes ``tests/golden/rlm/cases.json``: for every case the inputs' recipe (or
the explicit data), per-PE output hashes (keys, origins), per-level cut
matrices captured from ``mlpsort.rlm._cut_points`` (rlm.py:53-83), member
sizes after every level and the level reports (rlm.py:118-131).
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys

import numpy as np

from . import reference_loader

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden", "rlm", "cases.json")


def sha(values, dtype) -> str:
    return hashlib.sha256(np.asarray(list(values), dtype=dtype).tobytes()).hexdigest()


def run_case(name, data, p, groups, scheme, master_seed, stream, meta, store=False):
    reference_loader.load()
    from mlpsort import rlm
    from mlpsort.core import SeedSpec
    from mlpsort.simnet import Network

    levels: list = []
    orig = rlm._cut_points

    def wrapper(net, group, local, r, seed):
        members = list(group.members)
        cuts = orig(net, group, local, r, seed)
        lv = int(seed.stream_id.rsplit("/", 2)[1].split("-")[0][1:])
        while len(levels) <= lv:
            levels.append([])
        levels[lv].append({"group_lo": group.lo,
                           "sizes": [len(local[pe]) for pe in members],
                           "cuts": [[int(c) for c in cuts[pe]] for pe in members]})
        return cuts

    rlm._cut_points = wrapper
    rec = dict(meta)
    rec.update({"name": name, "p": p, "groups": list(groups), "scheme": scheme,
                "master_seed": master_seed, "stream": stream,
                "input_pe_sizes": [len(data[pe]) for pe in range(p)]})
    if store:
        rec["data"] = {str(pe): [int(e.key) for e in data[pe]] for pe in range(p)}
    try:
        try:
            plan = rlm.LevelPlan(p, tuple(groups))
            out, reports = rlm.rlm_sort(Network(p), data, plan, scheme, SeedSpec(master_seed, stream))
        except (ValueError, RuntimeError) as exc:
            rec["error"] = {"type": type(exc).__name__, "message": str(exc)}
            return rec
    finally:
        rlm._cut_points = orig
    offs = np.concatenate([[0], np.cumsum([len(data[pe]) for pe in range(p)])])
    flat = [e for pe in range(p) for e in out[pe]]
    rec.update({
        "input_sha256": sha((e.key for pe in range(p) for e in data[pe]), np.uint64),
        "output_sha256": sha((e.key for e in flat), np.uint64),
        "origin_sha256": sha((int(offs[e.origin_pe]) + e.origin_pos for e in flat), np.int64),
        "pe_sizes": [len(out[pe]) for pe in range(p)],
        "levels": levels,
        "reports": reports,
    })
    if store:
        rec["output"] = [[int(e.key), int(offs[e.origin_pe]) + e.origin_pos] for e in flat]
    return rec


def generated(dist, p, n_per_pe, seed):
    reference_loader.load()
    from mlpsort.bench import ExperimentConfig, generate_input
    return generate_input(ExperimentConfig(pes=p, n_per_pe=n_per_pe, dist=dist, seed=seed), 0)


def explicit(spec):
    reference_loader.load()
    from mlpsort.core import Element
    return {pe: [Element(k, pe, i) for i, k in enumerate(keys)] for pe, keys in spec.items()}


def cases():
    out = []
    for scheme in ("simple", "deterministic", "permuted", "randomized"):
        for dist in ("uniform", "sorted", "reverse", "equal", "zipf:1.1"):
            for groups, p in (((4, 4), 16), ((2, 2, 4), 16), ((16,), 16), ((8, 2), 16)):
                if scheme in ("permuted", "randomized") and (dist == "reverse" or groups == (16,)):
                    continue
                tag = f"{scheme}_{dist.replace(':', '')}_" + "x".join(map(str, groups))
                out.append((tag, lambda dist=dist, p=p, groups=groups, scheme=scheme, tag=tag: run_case(
                    tag, generated(dist, p, 200, 5), p, groups, scheme, 5, "algo/rep0",
                    {"dist": dist, "n_per_pe": 200, "input_seed": 5})))
    # BASELINE config shapes at reduced n.
    for name, dist, p, npe, groups, seed, scheme in (
            ("cfg1_scaled", "uniform", 16, 4096, (16,), 0, "deterministic"),
            ("cfg2_scaled", "uniform", 64, 1024, (8, 8), 1, "simple"),
            ("cfg2_scaled_det", "uniform", 64, 1024, (8, 8), 1, "deterministic"),
            ("cfg3_scaled", "uniform", 256, 128, (8, 32), 2, "simple"),
            ("cfg4_scaled_equal", "equal", 256, 64, (8, 32), 4, "simple"),
            ("cfg4_scaled_zipf", "zipf:1.1", 256, 64, (8, 32), 4, "deterministic")):
        out.append((name, lambda name=name, dist=dist, p=p, npe=npe, groups=groups, seed=seed,
                    scheme=scheme: run_case(name, generated(dist, p, npe, seed), p, groups, scheme,
                                            seed, "algo/rep0",
                                            {"dist": dist, "n_per_pe": npe, "input_seed": seed})))

    def tiny(name, spec, groups, scheme="simple", seed=9):
        out.append((name, lambda: run_case(name, explicit(spec), len(spec), groups, scheme, seed,
                                           "root", {"dist": "explicit"}, store=True)))

    # test_rlm.py shapes: one PE, ragged and empty PEs, fewer elements than parts, duplicates.
    tiny("tiny_single_pe", {0: [5, 3, 9, 1, 1, 0, 7, 3, 2, 8]}, (1,))
    tiny("tiny_empty_pes", {0: [3], 1: [], 2: [1], 3: []}, (2, 2))
    tiny("tiny_all_empty", {0: [], 1: [], 2: [], 3: []}, (4,))
    tiny("tiny_duplicates", {pe: [7] * 33 for pe in range(4)}, (2, 2), seed=7)
    rng = random.Random(77)
    tiny("tiny_ragged", {pe: [rng.randrange(50) for _ in range(rng.randrange(0, 40))]
                         for pe in range(8)}, (2, 4), seed=3)
    rng = random.Random(77)
    tiny("tiny_ragged_det", {pe: [rng.randrange(50) for _ in range(rng.randrange(0, 40))]
                             for pe in range(8)}, (2, 4), scheme="deterministic", seed=3)
    rng = random.Random(10)
    tiny("tiny_p6", {pe: [rng.randrange(1 << 20) for _ in range(30)] for pe in range(6)}, (3, 2), seed=12)
    tiny("tiny_fewer_than_parts", {0: [4, 2], 1: [], 2: [9], 3: [], 4: [], 5: [], 6: [], 7: []}, (8,))
    # One PE holds almost everything: pieces above ceil(n/p) (delivery.py:212-217).
    tiny("tiny_big_piece_det", {0: list(range(100)), 1: [5], 2: [7], 3: [9]}, (2, 2),
         scheme="deterministic", seed=2)
    tiny("tiny_big_piece_simple", {0: list(range(100)), 1: [5], 2: [7], 3: [9]}, (2, 2), seed=2)
    return out


def main(argv):
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    recs = []
    for name, build in cases():
        rec = build()
        recs.append(rec)
        print(name, "error" if "error" in rec else rec["pe_sizes"][:4])
    with open(OUT, "w") as f:
        json.dump(recs, f, separators=(",", ":"))
    print(f"{len(recs)} cases -> {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main(sys.argv[1:])
