"""Generate golden fixtures by running the REAL reference — TEST INFRA ONLY.

Runs ``mlpsort.ams.ams_sort`` (scheme ``"simple"``) from the read-only
``/root/reference`` on seeded inputs and records, per level and group, the
splitters (as ``(key, position-in-group-buffer)``), the global histogram,
the plan and the new member sizes, plus hashes of the final output and of
the origin permutation.  Output: ``tests/golden/<case>.json``.

    python oracle/make_goldens.py            # all cases
    python oracle/make_goldens.py cfg1 tiny  # selected cases

The fixtures travel with the repo; the GPU box never needs the reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import reference_loader  # noqa: E402

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def sha_u64(values) -> str:
    return hashlib.sha256(np.asarray(values, dtype="<u8").tobytes()).hexdigest()


def sha_i64(values) -> str:
    return hashlib.sha256(np.asarray(values, dtype="<i8").tobytes()).hexdigest()


def run_case(name, data, p, groups, a, b, eps, master_seed, stream, meta,
             store_data=False, scheme="simple"):
    mp = reference_loader.load()
    from mlpsort import ams
    from mlpsort.core import SeedSpec
    from mlpsort.simnet import Network

    levels: list = []
    orig_level = ams.ams_level
    orig_sel = ams.select_splitters
    orig_plan = ams.optimal_group_plan

    def level_wrapper(net, group, local, r, params, a_, scheme, seed):
        members = list(group.members)
        local_before_level = {pe: list(local[pe]) for pe in members}
        buf = [e for pe in members for e in local[pe]]
        index = {e: i for i, e in enumerate(buf)}
        cap = {}

        def sel(net_, group_, sample, buckets):
            s = orig_sel(net_, group_, sample, buckets)
            cap["splitters"] = s
            cap["bucket_count"] = buckets
            return s

        def plan(sizes, r_):
            pl = orig_plan(sizes, r_)
            cap["hist"] = [int(x) for x in sizes]
            cap["plan"] = pl
            return pl

        ams.select_splitters = sel
        ams.optimal_group_plan = plan
        try:
            rep = orig_level(net, group, local, r, params, a_, scheme, seed)
        finally:
            ams.select_splitters = orig_sel
            ams.optimal_group_plan = orig_plan
        pl = cap["plan"]
        lv = int(seed.stream_id.rsplit("/", 1)[1].split("-")[0][1:])
        while len(levels) <= lv:
            levels.append([])
        levels[lv].append({
            "group_lo": group.lo,
            "stream": seed.stream_id,
            "sizes": [len(local_before_level[pe]) for pe in members],
            "n_g": len(buf),
            "sample_size": rep["sample_size"],
            "bucket_count": rep["bucket_count"],
            "splitter_keys": [int(s.key) for s in cap["splitters"]],
            "splitter_pos": [index[s] for s in cap["splitters"]],
            "global_hist": cap["hist"],
            "boundaries": list(pl.boundaries),
            "loads": list(pl.loads),
            "max_load": pl.max_load,
            "load_budget": rep["load_budget"],
            "over_budget": bool(rep["over_budget"]),
            "new_sizes": [len(local[pe]) for pe in members],
        })
        return rep

    ams.ams_level = level_wrapper
    try:
        net = Network(p)
        params = ams.AmsParams(tuple(groups), oversampling=a,
                               overpartition=b, imbalance=eps)
        seed = SeedSpec(master_seed, stream)
        t0 = time.perf_counter()
        try:
            out, reports = ams.ams_sort(net, data, params, scheme, seed)
        except (ValueError, RuntimeError) as exc:
            # The reference rejects this input (e.g. deliver_deterministic's
            # piece bound, delivery.py:212-217): the fixture pins the error.
            rec = dict(meta)
            rec.update({"name": name, "p": p, "groups": list(groups), "a": a, "b": b,
                        "eps": eps, "master_seed": master_seed, "stream": stream,
                        "scheme": scheme, "input_pe_sizes": [len(data[pe]) for pe in range(p)],
                        "error": {"type": type(exc).__name__, "message": str(exc)}})
            if store_data:
                rec["data"] = {str(pe): [[int(e.key), e.origin_pe, e.origin_pos]
                                         for e in data[pe]] for pe in range(p)}
            return rec
        wall = time.perf_counter() - t0
    finally:
        ams.ams_level = orig_level
    offs = np.concatenate([[0], np.cumsum([len(data[pe]) for pe in range(p)])])
    flat = [e for pe in range(p) for e in out[pe]]
    in_keys = [e.key for pe in range(p) for e in data[pe]]
    rec = dict(meta)
    rec.update({
        "name": name, "p": p, "groups": list(groups), "a": a, "b": b,
        "eps": eps, "master_seed": master_seed, "stream": stream,
        "scheme": scheme,
        "input_pe_sizes": [len(data[pe]) for pe in range(p)],
        "input_sha256": sha_u64(in_keys),
        "output_sha256": sha_u64([e.key for e in flat]),
        "origin_sha256": sha_i64([int(offs[e.origin_pe]) + e.origin_pos for e in flat]),
        "pe_sizes": [len(out[pe]) for pe in range(p)],
        "levels": levels,
        "reports": [{k: (bool(v) if isinstance(v, bool) else v)
                     for k, v in r.items()} for r in reports],
        "reference_wall_s": wall,
    })
    if store_data:
        rec["data"] = {str(pe): [[int(e.key), e.origin_pe, e.origin_pos]
                                 for e in data[pe]] for pe in range(p)}
        rec["output"] = [[int(e.key), e.origin_pe, e.origin_pos] for e in flat]
    return rec


def generated(dist, p, n_per_pe, seed):
    reference_loader.load()
    from mlpsort.bench import ExperimentConfig, generate_input
    cfg = ExperimentConfig(pes=p, n_per_pe=n_per_pe, dist=dist, seed=seed)
    return generate_input(cfg, 0)


def explicit(spec):
    reference_loader.load()
    from mlpsort.core import Element
    return {pe: [Element(k, pe, i) for i, k in enumerate(keys)]
            for pe, keys in spec.items()}


def cases():
    """(name, builder) pairs; builders return the fixture dict."""
    out = []

    def cfg(name, dist, p, npe, groups, a, b, eps, seed, store=False, scheme="simple"):
        def build():
            data = generated(dist, p, npe, seed)
            meta = {"dist": dist, "n_per_pe": npe, "input_seed": seed}
            return run_case(name, data, p, groups, a, b, eps, seed, "algo/rep0",
                            meta, store_data=store, scheme=scheme)
        out.append((name, build))

    # SURVEY §8(d) config 1, full size.
    cfg("cfg1", "uniform", 16, 65536, (16,), 16.0, 16, 0.1, 0)
    # Configs 2 / 3 at reduced n (same p, group counts, a-rule, b, eps).
    cfg("cfg2_scaled", "uniform", 64, 1 << 14, (8, 8), None, 16, 0.1, 1)
    cfg("cfg3_scaled", "uniform", 256, 1 << 12, (8, 32), None, 16, 0.1, 2)
    # Config 5 shapes at the small end (pool-path sampling, k=1 vs k=2).
    cfg("cfg5_k1_small", "uniform", 256, 32, (256,), None, 16, 0.1, 3)
    cfg("cfg5_k2_small", "uniform", 256, 32, (8, 32), None, 16, 0.1, 3)
    # Distribution × schedule grid (SURVEY Appendix B-3/B-8 shapes).
    for dist in ("uniform", "sorted", "reverse", "equal", "zipf:1.1", "zipf:3"):
        for groups, p in (((4, 4), 16), ((2, 2, 4), 16), ((16,), 16), ((8, 2), 16)):
            tag = dist.replace(":", "") + "_" + "x".join(map(str, groups))
            cfg(f"dist_{tag}", dist, p, 250, groups, None, 8, 0.2, 5)
    # Skewed shapes at config-4 schedule, reduced n.
    for dist in ("sorted", "reverse", "equal", "zipf:1.1"):
        cfg(f"cfg4_scaled_{dist.replace(':', '')}", dist, 256, 256, (8, 32),
            None, 16, 0.1, 4)

    # deliver_deterministic (the CLI / bench default scheme, delivery.py:188-306):
    # it places members differently from "simple" on sorted / equal inputs.
    for dist in ("uniform", "sorted", "reverse", "equal", "zipf:1.1"):
        for groups, p in (((4, 4), 16), ((8, 2), 16), ((2, 2, 4), 16)):
            tag = dist.replace(":", "") + "_" + "x".join(map(str, groups))
            cfg(f"det_{tag}", dist, p, 250, groups, None, 8, 0.2, 5, scheme="deterministic")
    cfg("det_cfg2_scaled", "uniform", 64, 1 << 12, (8, 8), None, 16, 0.1, 1,
        scheme="deterministic")
    for dist in ("sorted", "equal"):
        cfg(f"det_cfg4_scaled_{dist}", dist, 256, 128, (8, 32), None, 16, 0.1, 4,
            scheme="deterministic")
        # at (8, 8) sorted / equal inputs place members differently.
        cfg(f"det_cfg2_scaled_{dist}", dist, 64, 1 << 12, (8, 8), None, 16, 0.1, 1,
            scheme="deterministic")
        cfg(f"simple_cfg2_scaled_{dist}", dist, 64, 1 << 12, (8, 8), None, 16, 0.1, 1)

    # deliver_simple_permuted (delivery.py:183-185): Feistel enumeration orders.
    for dist in ("uniform", "sorted", "equal", "zipf:1.1"):
        for groups, p in (((4, 4), 16), ((2, 2, 4), 16)):
            tag = dist.replace(":", "") + "_" + "x".join(map(str, groups))
            cfg(f"perm_{tag}", dist, p, 250, groups, None, 8, 0.2, 5, scheme="permuted")
    cfg("perm_cfg2_scaled_equal", "equal", 64, 1 << 12, (8, 8), None, 16, 0.1, 1,
        scheme="permuted")
    # deliver_randomized (delivery.py:318-436): chunking, delegation, shuffles.
    for dist in ("uniform", "sorted", "equal", "zipf:1.1"):
        for groups, p in (((4, 4), 16), ((2, 2, 4), 16), ((8, 2), 16)):
            tag = dist.replace(":", "") + "_" + "x".join(map(str, groups))
            cfg(f"rand_{tag}", dist, p, 250, groups, None, 8, 0.2, 5, scheme="randomized")
    cfg("rand_cfg2_scaled_sorted", "sorted", 64, 1 << 12, (8, 8), None, 16, 0.1, 1,
        scheme="randomized")
    cfg("perm_cfg3_scaled", "uniform", 256, 1 << 9, (8, 32), None, 16, 0.1, 2,
        scheme="permuted")

    def tiny(name, spec, groups, b=16, eps=0.2, seed=9, scheme="simple"):
        def build():
            data = explicit(spec)
            p = len(spec)
            return run_case(name, data, p, groups, None, b, eps, seed, "root",
                            {"dist": "explicit"}, store_data=True, scheme=scheme)
        out.append((name, build))

    # test_ams.py:292-299 shape, with scheme simple.
    tiny("tiny_empty_pes", {0: [3], 1: [], 2: [1], 3: []}, (2, 2))
    # test_ams.py:253-259 heavy duplicates.
    tiny("tiny_duplicates", {pe: [7] * 64 for pe in range(4)}, (2, 2), seed=7)
    # test_ams.py:146-154 non-power-of-two machine.
    import random as _r
    rng = _r.Random(10)
    tiny("tiny_p6", {pe: [rng.randrange(1 << 20) for _ in range(30)]
                     for pe in range(6)}, (3, 2), b=4, seed=12)
    tiny("tiny_single_pe", {0: [5, 3, 9, 1, 1, 0, 7, 3, 2, 8, 6, 4]}, (1,), seed=1)
    rng = _r.Random(77)
    tiny("tiny_ragged", {pe: [rng.randrange(50) for _ in range(rng.randrange(0, 40))]
                         for pe in range(8)}, (2, 4), b=4, seed=3)
    rng = _r.Random(77)
    tiny("det_tiny_ragged", {pe: [rng.randrange(50) for _ in range(rng.randrange(0, 40))]
                             for pe in range(8)}, (2, 4), b=4, seed=3, scheme="deterministic")
    rng = _r.Random(5)
    tiny("det_tiny_mixed", {pe: [rng.randrange(1 << 30) for _ in range(20 + 3 * pe)]
                            for pe in range(8)}, (2, 4), b=4, seed=8, scheme="deterministic")
    rng = _r.Random(6)
    tiny("perm_tiny_ragged", {pe: [rng.randrange(60) for _ in range(rng.randrange(0, 30))]
                              for pe in range(8)}, (2, 4), b=4, seed=4, scheme="permuted")
    rng = _r.Random(8)
    tiny("rand_tiny_ragged", {pe: [rng.randrange(60) for _ in range(rng.randrange(0, 30))]
                              for pe in range(8)}, (2, 4), b=4, seed=4, scheme="randomized")
    # One big PE: its piece exceeds ceil(n/p) (delivery.py:212-217 ValueError).
    tiny("det_tiny_big_piece", {0: list(range(100)), 1: [5], 2: [7], 3: [9]}, (2, 2), b=4,
         seed=2, scheme="deterministic")
    return out


def main(argv):
    os.makedirs(GOLDEN_DIR, exist_ok=True)
    want = set(argv)
    for name, build in cases():
        if want and name not in want and not any(name.startswith(w) for w in want):
            continue
        t0 = time.perf_counter()
        rec = build()
        path = os.path.join(GOLDEN_DIR, f"{name}.json")
        with open(path, "w") as f:
            json.dump(rec, f, separators=(",", ":"))
        print(f"{name}: {time.perf_counter() - t0:.1f}s -> {path}")


if __name__ == "__main__":
    main(sys.argv[1:])
