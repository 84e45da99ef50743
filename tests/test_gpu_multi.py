"""Single-process multi-device driver (ams_mg_sort_run) on
ONE GPU: G contexts on device 0 run the same code path as G devices (the
level-1 scatter stores through the owners' buffer pointers; the host
synchronises the contexts, no kernel waits on another).  Results must be
bit-identical to the oracle for every G."""

import numpy as np
import pytest

from oracle import ams_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _input(groups, npe, dist_kind, seed=4):
    p = int(np.prod(groups))
    n = p * npe
    rng = np.random.default_rng(seed)
    keys = {"uniform": lambda: rng.integers(0, 2**64, n, dtype=np.uint64),
            "zipf": lambda: O.zipf_keys(n, 3), "sorted": lambda: np.arange(n, dtype=np.uint64),
            "equal": lambda: np.full(n, 7, dtype=np.uint64)}[dist_kind]()
    return keys, [npe] * p


def run_mg(G, keys, sizes, groups, scheme="simple", with_vals=False, eps=0.1):
    from paper_1410_6754_b200 import AmsParams, SeedSpec
    from paper_1410_6754_b200.multi import MultiDeviceSorter
    p = len(sizes)
    pl = p // G
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    ks = [torch.from_numpy(keys[offs[i * pl]:offs[(i + 1) * pl]].view(np.int64).copy()).cuda() for i in range(G)]
    vs = [torch.arange(int(offs[i * pl]), int(offs[(i + 1) * pl]), dtype=torch.int64, device="cuda")
          for i in range(G)] if with_vals else None
    mg = MultiDeviceSorter([0] * G)
    try:
        outs = []
        for _ in range(2):  # the second run reuses every buffer
            ok, ov, sz, reports, l1 = mg.sort(ks, sizes, AmsParams(tuple(groups), None, 16, eps),
                                              SeedSpec(5, "algo/rep0"), vals=vs, scheme=scheme, key_kind="u64")
            later = []
            for i in range(G):
                ctx = mg.context(i)
                later.append([[[int(x) for x in row] for row in ctx.run_level(lv)["boundaries"]]
                              for lv in range(1, len(groups))])
            outs.append((np.concatenate([t.cpu().numpy().view(np.uint64) for t in ok]),
                         None if ov is None else np.concatenate([t.cpu().numpy() for t in ov]),
                         [int(x) for x in sz], reports, l1, later))
        return outs
    finally:
        mg.close()


def _ref_later(ref, G, i):
    out = []
    for infos in ref.levels[1:]:
        per = len(infos) // G
        out.append([list(x.plan.boundaries) for x in infos[i * per:(i + 1) * per]])
    return out


@pytest.mark.parametrize("G", [1, 2, 4])
@pytest.mark.parametrize("groups,npe,dist_kind,with_vals", [
    ((8, 8), 3000, "uniform", True), ((8, 8), 3000, "uniform", False), ((4, 4), 5000, "zipf", True),
    ((8,), 9000, "sorted", False), ((4, 2, 2), 2500, "equal", True),
])
def test_mg_simple_matches_oracle(G, groups, npe, dist_kind, with_vals):
    keys, sizes = _input(groups, npe, dist_kind)
    n = len(keys)
    ref = O.ams_sort(keys, sizes, groups, None, 16, 0.1, 5, "algo/rep0",
                     vals=np.arange(n, dtype=np.int64) if with_vals else None)
    for out, ov, sz, reports, l1, later in run_mg(G, keys, sizes, groups, "simple", with_vals):
        assert np.array_equal(out, ref.keys)
        if with_vals:
            assert np.array_equal(ov, ref.vals)
        assert sz == list(ref.pe_sizes)
        assert [int(x) for x in l1["boundaries"]] == list(ref.levels[0][0].plan.boundaries)
        assert np.array_equal(l1["seg_hist"][:, :ref.levels[0][0].hist.shape[1]], ref.levels[0][0].hist)
        for i in range(G):
            assert later[i] == _ref_later(ref, G, i)
        for mine, theirs in zip(reports, ref.reports):
            for key, v in theirs.items():
                assert mine[key] == int(v), (key, mine[key], v)


@pytest.mark.parametrize("G", [1, 2])
@pytest.mark.parametrize("scheme", ["deterministic", "permuted", "randomized"])
@pytest.mark.parametrize("groups,npe,dist_kind", [
    ((4, 4), 3000, "sorted"), ((8, 8), 2000, "uniform"), ((2, 2, 4), 2500, "zipf"), ((16,), 4000, "uniform"),
])
def test_mg_other_schemes_match_oracle(G, scheme, groups, npe, dist_kind):
    keys, sizes = _input(groups, npe, dist_kind)
    ref = O.ams_sort(keys, sizes, groups, None, 16, 0.1, 5, "algo/rep0", scheme=scheme)
    for out, _, sz, reports, l1, later in run_mg(G, keys, sizes, groups, scheme):
        assert np.array_equal(out, ref.keys)
        assert sz == list(ref.pe_sizes)
        assert [int(x) for x in l1["boundaries"]] == list(ref.levels[0][0].plan.boundaries)
        assert [int(x) for x in l1["new_sizes"]] == list(ref.levels[0][0].new_sizes)
        for i in range(G):
            assert later[i] == _ref_later(ref, G, i)
        for mine, theirs in zip(reports, ref.reports):
            for key, v in theirs.items():
                assert mine[key] == int(v), (key, mine[key], v)


def test_mg_cfg3_shape_scaled():
    """Config 3's shape (p=256, (8,32), f64 in [0,1)) at reduced n on 1/2/4/8
    contexts: the same bits for every G."""
    from paper_1410_6754_b200 import AmsParams, SeedSpec
    from paper_1410_6754_b200.multi import MultiDeviceSorter
    p, npe = 256, 2048
    x = np.random.default_rng(2).random(p * npe)
    ref = O.ams_sort(O.f64_to_ordered_u64(x), [npe] * p, (8, 32), None, 16, 0.1, 2, "algo/rep0")
    for G in (1, 2, 4, 8):
        pl = p // G
        ks = [torch.from_numpy(x[i * pl * npe:(i + 1) * pl * npe].copy()).cuda() for i in range(G)]
        mg = MultiDeviceSorter([0] * G)
        try:
            ok, _, sz, reports, l1 = mg.sort(ks, [npe] * p, AmsParams((8, 32), None, 16, 0.1),
                                             SeedSpec(2, "algo/rep0"), key_kind="f64")
        finally:
            mg.close()
        out = np.concatenate([t.cpu().numpy() for t in ok])
        assert np.array_equal(out, np.sort(x))
        assert [int(v) for v in sz] == list(ref.pe_sizes)
        assert [int(v) for v in l1["boundaries"]] == list(ref.levels[0][0].plan.boundaries)


def test_mg_rejects_bad_shapes():
    from paper_1410_6754_b200 import AmsParams, SeedSpec
    from paper_1410_6754_b200.multi import MultiDeviceSorter
    mg = MultiDeviceSorter([0, 0, 0, 0])
    try:
        ks = [torch.zeros(16, dtype=torch.int64, device="cuda") for _ in range(4)]
        with pytest.raises(ValueError, match="multiple of the 4 devices"):
            mg.sort(ks, [8] * 8, AmsParams((2, 4), None, 16, 0.1), SeedSpec(1, "x"))
        with pytest.raises(ValueError, match="simple delivery scheme only"):
            mg.sort(ks, [8] * 8, AmsParams((4, 2), None, 16, 0.1), SeedSpec(1, "x"), vals=ks,
                    scheme="deterministic")
    finally:
        mg.close()


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("scheme", ["simple", "deterministic"])
def test_mg_ragged_and_empty_contexts(G, scheme):
    """Ragged PE sizes, PEs without keys, and a whole context without input
    (it still receives its groups' keys)."""
    from paper_1410_6754_b200 import AmsParams, SeedSpec
    from paper_1410_6754_b200.multi import MultiDeviceSorter
    groups, p = (4, 4), 16
    rng = np.random.default_rng(G * 3 + len(scheme))
    sizes = [int(x) for x in rng.integers(0, 3000, p)]
    sizes[1] = 0
    for j in range(p // G):          # the first context holds nothing
        sizes[j] = 0
    n = sum(sizes)
    keys = rng.integers(0, 1 << 40, n, dtype=np.uint64)
    ref = O.ams_sort(keys, sizes, groups, None, 16, 0.3, 5, "algo/rep0", scheme=scheme)
    pl = p // G
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    ks = [torch.from_numpy(keys[offs[i * pl]:offs[(i + 1) * pl]].view(np.int64).copy()).cuda() for i in range(G)]
    mg = MultiDeviceSorter([0] * G)
    try:
        ok, _, sz, reports, l1 = mg.sort(ks, sizes, AmsParams(groups, None, 16, 0.3), SeedSpec(5, "algo/rep0"),
                                         scheme=scheme, key_kind="u64")
    finally:
        mg.close()
    out = np.concatenate([t.cpu().numpy().view(np.uint64) for t in ok])
    assert np.array_equal(out, ref.keys)
    assert [int(x) for x in sz] == list(ref.pe_sizes)
    assert [int(x) for x in l1["boundaries"]] == list(ref.levels[0][0].plan.boundaries)


def test_mg_empty_input():
    from paper_1410_6754_b200 import AmsParams, SeedSpec
    from paper_1410_6754_b200.multi import MultiDeviceSorter
    mg = MultiDeviceSorter([0, 0])
    try:
        ks = [torch.zeros(0, dtype=torch.int64, device="cuda") for _ in range(2)]
        ok, _, sz, reports, _ = mg.sort(ks, [0] * 8, AmsParams((4, 2), None, 16, 0.1), SeedSpec(1, "x"),
                                        key_kind="u64")
    finally:
        mg.close()
    assert all(t.numel() == 0 for t in ok) and [int(x) for x in sz] == [0] * 8
