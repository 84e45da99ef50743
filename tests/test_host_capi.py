"""CPU tests of the C ABI's host helpers (no GPU): the seeded-stream
restatement (blake2b -> MT19937 -> random.sample), the grouping plan, the
level planner, and that the library exports every symbol the header
declares."""

import hashlib
import random
import re

import numpy as np
import pytest

from oracle import ams_oracle as O
from paper_1410_6754_b200 import _lib as L
from tests import golden_util as G


def test_header_symbols_exported():
    text = open("include/ams_b200.h").read()
    declared = set(re.findall(r"^\s*(?:int|uint64_t|const char\*)\s+(ams_\w+)\(", text, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(L.EXPORTED), declared ^ set(L.EXPORTED)
    for name in declared:
        assert hasattr(L.lib, name)


@pytest.mark.parametrize("n", [0, 1, 15, 127, 128, 129, 255, 256, 300])
def test_blake2b_matches_hashlib(n):
    msg = bytes((i * 37 + 11) & 0xFF for i in range(n))
    assert L.blake2b_128(msg) == hashlib.blake2b(msg, digest_size=16).digest()


@pytest.mark.parametrize("stream", ["root", "algo/rep0/L0-g0/sample/pe5", "input/rep0/pe15", "x" * 200])
@pytest.mark.parametrize("master", [0, 1, 8042, 123456789])
def test_stream_seed_words(master, stream):
    x = O.stream_seed_int(master, stream)
    words = L.stream_seed_words(master, stream)
    nw = max(1, (x.bit_length() + 31) // 32)
    assert len(words) == nw
    assert sum(int(w) << (32 * i) for i, w in enumerate(words)) == x


def _words(x):
    n = max(1, (x.bit_length() + 31) // 32)
    return np.array([(x >> (32 * i)) & 0xFFFFFFFF for i in range(n)], dtype=np.uint32)


@pytest.mark.parametrize("x", [0, 1, 2**32, 2**96 - 5, 2**128 - 1,
                               O.stream_seed_int(0, "algo/rep0/L0-g0/sample/pe0")])
@pytest.mark.parametrize("k", [1, 7, 31, 32, 33, 53, 64])
def test_getrandbits_matches_cpython(x, k):
    rng = random.Random(x)
    want = [rng.getrandbits(k) for _ in range(300)]
    got = L.getrandbits(_words(x), k, 300)
    assert [int(v) for v in got] == want


@pytest.mark.parametrize("k", [32, 64])
def test_getrandbits_across_state_twists(k):
    # 64-bit draws use two words: 5000 draws run through 16 twists of the
    # 624-word state, which the library regenerates one word at a time.
    x = O.stream_seed_int(3, "algo/rep0/L1-g8/sample/pe9")
    rng = random.Random(x)
    want = [rng.getrandbits(k) for _ in range(5000)]
    got = L.getrandbits(_words(x), k, 5000)
    assert [int(v) for v in got] == want


@pytest.mark.parametrize("n,k", [(32, 32), (65536, 256), (1 << 22, 231), (100, 40), (1 << 27, 9),
                                 (10, 0), (1, 1), (5, 5), (6, 6), (21, 5), (22, 6), (5000, 1727),
                                 (16405, 1727), (16406, 1727), (3, 2), (1 << 31, 100)])
def test_sample_matches_cpython(n, k):
    for seed in (0, 7, O.stream_seed_int(3, "algo/rep0/L1-g8/sample/pe9")):
        want = sorted(random.Random(seed).sample(range(n), k))
        got = L.sample_indices(_words(seed), n, k)
        assert [int(v) for v in got] == want


def test_sample_rejects_oversized():
    with pytest.raises(ValueError):
        L.sample_indices(_words(1), 3, 4)


def test_draw_sample_positions_matches_oracle():
    sizes = np.array([40, 0, 3, 100, 17, 64, 64, 5], dtype=np.uint64)
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.uint64)
    gf, gn = np.array([0, 4], np.int32), np.array([4, 4], np.int32)
    targets = np.array([60, 100], np.uint64)
    idx, gpos, cnt = L.draw_sample_positions(5, "algo/rep0", 1, gf, gn, targets, sizes, offs)
    w = 0
    for g in range(2):
        base, extra = divmod(int(targets[g]), int(gn[g]))
        gp = 0
        for i in range(int(gn[g])):
            pe = int(gf[g]) + i
            take = min(base + (i < extra), int(sizes[pe]))
            want = O.sample_indices(5, f"algo/rep0/L1-g{int(gf[g])}/sample/pe{pe}", int(sizes[pe]), take)
            assert [int(v) for v in idx[w:w + take]] == [int(offs[pe]) + t for t in want]
            assert [int(v) for v in gpos[w:w + take]] == [gp + t for t in want]
            w += take
            gp += int(sizes[pe])
    assert w == len(idx) == int(cnt.sum())


def test_plan_hand_cases():
    assert L.scan_groups([5, 3, 4, 2, 6], 3, 8) == ((0, 2, 4, 5), (8, 6, 6), 8)
    assert L.scan_groups([5, 3, 4, 2, 6], 3, 7) is None
    assert L.scan_groups([5, 3, 4], 3, 5)[1] == (5, 3, 4)
    assert L.scan_groups([5, 3], 2, 4) is None
    assert L.group_plan([5, 3, 4, 2, 6], 3)[2] == 8
    assert L.group_plan([5, 3, 4, 2, 6], 1)[2] == 20
    assert L.group_plan([5, 3, 4, 2, 6], 7)[2] == 6
    assert L.group_plan([0, 0, 0], 2)[2] == 0


def test_plan_matches_oracle_random():
    rng = np.random.default_rng(0)
    for _ in range(3000):
        nb = int(rng.integers(1, 300))
        r = int(rng.integers(1, 40))
        mode = rng.integers(0, 3)
        hi = [6, 1000, 5][mode]
        sizes = rng.integers(0, hi, nb)
        if mode == 2:
            sizes[rng.random(nb) < 0.5] = 0
        want = O.group_plan(sizes.tolist(), r)
        got = L.group_plan(sizes, r)
        assert got == (want.boundaries, want.loads, want.max_load)


@pytest.mark.parametrize("name", ["cfg2_scaled", "cfg3_scaled", "dist_zipf1.1_2x2x4",
                                  "tiny_empty_pes", "cfg4_scaled_sorted", "cfg5_k1_small"])
def test_plan_level_matches_golden(name):
    """Given the oracle's per-member histograms, the native planner gives
    the reference's plans, next-level sizes and exchange stats."""
    g = G.load(name)
    keys, sizes = G.input_of(g)
    res = O.ams_sort(keys, sizes, tuple(g["groups"]), g["a"], g["b"], g["eps"],
                     g["master_seed"], g["stream"])
    for lv, infos in enumerate(res.levels):
        r = g["groups"][lv]
        nb_stride = max(i.bucket_count for i in infos)
        hist = np.zeros((sum(i.hist.shape[0] for i in infos), nb_stride), np.uint32)
        row = 0
        for i in infos:
            hist[row:row + i.hist.shape[0], :i.hist.shape[1]] = i.hist
            row += i.hist.shape[0]
        gn = [i.hist.shape[0] for i in infos]
        nb = [i.bucket_count for i in infos]
        bnd, loads, mx, new_sizes, stats = L.plan_level(gn, nb, r, hist)
        row = 0
        for gi, (info, ref) in enumerate(zip(infos, g["levels"][lv])):
            assert [int(x) for x in bnd[gi]] == ref["boundaries"]
            assert [int(x) for x in loads[gi]] == ref["loads"]
            assert int(mx[gi]) == ref["max_load"]
            P = info.hist.shape[0]
            assert [int(x) for x in new_sizes[row:row + P]] == ref["new_sizes"]
            assert [int(x) for x in stats[gi]] == [info.stats[k] for k in
                                                   ("max_words", "max_msgs", "max_sent_msgs",
                                                    "max_recv_msgs")]
            row += P


def test_errors_map_to_valueerror():
    with pytest.raises(ValueError):
        L.group_plan([1, 2], 0)
    with pytest.raises(ValueError):
        L.plan_level([3], [4], 2, np.zeros((3, 4), np.uint32))  # 3 PEs cannot form 2 groups


def test_deterministic_delivery_matches_oracle_random():
    """The native deliver_deterministic assignment (delivery.py:188-306)
    equals the oracle's restatement: sizes, receive-order layout, exchange
    stats and the reference's error messages."""
    rng = np.random.default_rng(0)
    for trial in range(600):
        r, sub = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        P = r * sub
        if trial % 3 == 0:
            pcs = rng.integers(0, 50, (P, r))
        elif trial % 3 == 1:
            pcs = rng.integers(0, 3, (P, r)) * rng.integers(0, 100, (P, r))
        else:
            pcs = np.zeros((P, r), np.int64)
            for j in range(P):
                pcs[j, rng.integers(0, r)] = rng.integers(0, 40)
        try:
            slices, sizes = O.deterministic_plan(pcs.astype(np.int64), 3)
            err = None
        except (ValueError, RuntimeError) as e:
            err = (type(e), str(e))
        if err:
            with pytest.raises(err[0], match=re.escape(err[1])):
                L.deliver_deterministic(pcs, 3)
            continue
        ns, sl, st = L.deliver_deterministic(pcs, 3)
        assert [int(x) for x in ns] == sizes
        e_layout = np.arange(int(pcs.sum()))
        want = O.deterministic_relayout(e_layout, pcs.astype(np.int64), slices, sizes)
        got = np.empty_like(e_layout)
        for s0, d0, ln in sl:
            got[int(d0):int(d0 + ln)] = e_layout[int(s0):int(s0 + ln)]
        assert np.array_equal(got, want)
        ref = O._deterministic_stats(pcs.astype(np.int64), slices)
        assert [int(x) for x in st] == [ref[k] for k in ("max_words", "max_msgs", "max_sent_msgs",
                                                         "max_recv_msgs")]


@pytest.mark.parametrize("name", ["det_cfg2_scaled_equal", "det_reverse_2x2x4", "det_tiny_mixed"])
def test_deterministic_delivery_matches_golden(name):
    """Piece sizes from the oracle's level histograms and plans -> the native
    assignment gives the reference's new member sizes (golden fixtures)."""
    g = G.load(name)
    keys, sizes = G.input_of(g)
    res = O.ams_sort(keys, sizes, tuple(g["groups"]), g["a"], g["b"], g["eps"],
                     g["master_seed"], g["stream"], scheme="deterministic")
    for lv, infos in enumerate(res.levels):
        r = g["groups"][lv]
        for info, ref in zip(infos, g["levels"][lv]):
            bnd = info.plan.boundaries
            pcs = np.stack([info.hist[:, bnd[t]:bnd[t + 1]].sum(axis=1) for t in range(r)], axis=1)
            ns, _, _ = L.deliver_deterministic(pcs, info.group_lo)
            assert [int(x) for x in ns] == ref["new_sizes"]


@pytest.mark.parametrize("scheme", ["permuted", "randomized"])
def test_seeded_delivery_matches_oracle_random(scheme):
    """The native deliver_simple_permuted (Feistel enumeration,
    delivery.py:151-185, core.py:96-159) and deliver_randomized (chunking,
    delegation, CPython shuffles, delivery.py:318-436) slices equal the
    oracle's restatements."""
    planner, native = {"permuted": (O.permuted_plan, L.deliver_permuted),
                       "randomized": (O.randomized_plan, L.deliver_randomized)}[scheme]
    rng = np.random.default_rng(1)
    for trial in range(300):
        r, sub = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        P = r * sub
        pcs = rng.integers(0, 40, (P, r)) * (rng.random((P, r)) < 0.7)
        if trial % 4 == 0:
            pcs[0, 0] = 400  # one large piece: chunked and delegated
        ls = f"algo/rep0/L{trial % 3}-g{trial % 7}"
        slices, sizes = planner(pcs.astype(np.int64), 5, ls)
        ns, sl, st = native(pcs, 5, ls)
        assert [int(x) for x in ns] == sizes
        e_layout = np.arange(int(pcs.sum()))
        want = O.deterministic_relayout(e_layout, pcs.astype(np.int64), slices, sizes)
        got = np.empty_like(e_layout)
        for s0, d0, ln in sl:
            got[int(d0):int(d0 + ln)] = e_layout[int(s0):int(s0 + ln)]
        assert np.array_equal(got, want)
        ref = O._deterministic_stats(pcs.astype(np.int64), slices)
        assert [int(x) for x in st] == [ref[k] for k in ("max_words", "max_msgs", "max_sent_msgs",
                                                         "max_recv_msgs")]
