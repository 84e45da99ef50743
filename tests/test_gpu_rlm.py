"""GPU parity of RLM-sort through the C ABI
(``ams_rlm_sort_run``): golden fixtures from the real reference
(rlm.py:86-132) and the CPU oracle at sizes the reference cannot reach."""

import numpy as np
import pytest

from tests import rlm_golden_util as RG

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def run_gpu(keys, sizes, groups, scheme, seed, stream, vals=None, kind="u64"):
    from paper_1410_6754_b200 import LevelPlan, SeedSpec, rlm_sort_tensors
    view = keys.view(np.int64) if keys.dtype == np.uint64 else keys
    d_keys = torch.from_numpy(np.ascontiguousarray(view)).cuda()
    d_vals = None if vals is None else torch.from_numpy(vals).cuda()
    res = rlm_sort_tensors(d_keys, sizes, LevelPlan(len(sizes), tuple(groups)), SeedSpec(seed, stream),
                           vals=d_vals, scheme=scheme, key_kind=kind)
    torch.cuda.synchronize()
    return res


def level_views(res):
    cuts, sizes_after = [], []
    for d in res.levels:
        per_group = []
        for gf, gn in zip(d["group_first"], d["group_npe"]):
            per_group.append(d["cuts"][gf:gf + gn].astype(np.int64))
        cuts.append(per_group)
        sizes_after.append(d["new_sizes"])
    return cuts, sizes_after


@pytest.mark.parametrize("name", RG.NAMES)
def test_rlm_golden_parity(name):
    g = RG.CASES[name]
    keys, sizes = RG.input_of(g)
    if "error" in g:
        exc = {"ValueError": ValueError, "RuntimeError": RuntimeError}[g["error"]["type"]]
        with pytest.raises(exc) as ei:
            run_gpu(keys, sizes, g["groups"], g["scheme"], g["master_seed"], g["stream"])
        assert g["error"]["message"] in str(ei.value)
        return
    res = run_gpu(keys, sizes, g["groups"], g["scheme"], g["master_seed"], g["stream"])
    cuts, sizes_after = level_views(res)
    RG.check(g, keys, res.keys.cpu().numpy().view(np.uint64), res.origin.cpu().numpy(), res.pe_sizes,
             cuts, sizes_after, res.reports)
    assert res.launches > 0 or len(keys) == 0


@pytest.mark.parametrize("scheme", ["simple", "deterministic", "permuted", "randomized"])
@pytest.mark.parametrize("p,groups,npe,bits", [(64, (8, 8), 4096, 64), (64, (4, 4, 4), 1500, 10),
                                               (32, (32,), 9000, 64), (16, (2, 8), 20000, 3)])
def test_rlm_oracle_parity(scheme, p, groups, npe, bits):
    from oracle import rlm_oracle as R
    rng = np.random.default_rng(p * 1000 + npe + bits)
    sizes = [int(x) for x in rng.integers(max(1, npe - 50), npe + 1, p)]   # near-equal, ragged
    n = sum(sizes)
    keys = rng.integers(0, 2**bits if bits < 64 else 2**64, n, dtype=np.uint64)
    vals = rng.integers(0, 2**62, n, dtype=np.int64)
    ref = R.rlm_sort(keys, sizes, groups, scheme, 11, "t/rep0", vals=vals)
    res = run_gpu(keys, sizes, groups, scheme, 11, "t/rep0", vals=vals)
    assert np.array_equal(res.keys.cpu().numpy().view(np.uint64), ref.keys)
    assert np.array_equal(res.origin.cpu().numpy(), ref.origin)
    assert np.array_equal(res.vals.cpu().numpy(), ref.vals)
    assert [int(x) for x in res.pe_sizes] == list(ref.pe_sizes)
    for d, infos in zip(res.levels, ref.levels):
        for info, gf, gn in zip(infos, d["group_first"], d["group_npe"]):
            assert np.array_equal(d["cuts"][gf:gf + gn].astype(np.int64), info.cuts)
    for mine, theirs in zip(res.reports, ref.reports):
        assert mine == theirs
    # perfect balance (rlm.py:1-9): parts differ by at most one element per level
    assert max(res.pe_sizes) - min(res.pe_sizes) <= len(groups) + 1


def test_rlm_f64_and_i64_keys():
    from oracle import ams_oracle as O, rlm_oracle as R
    rng = np.random.default_rng(5)
    p, npe = 16, 3000
    x = rng.standard_normal(p * npe)
    ref = R.rlm_sort(O.f64_to_ordered_u64(x), [npe] * p, (4, 4), "simple", 3, "f")
    res = run_gpu(x, [npe] * p, (4, 4), "simple", 3, "f", kind="f64")
    assert np.array_equal(res.keys.cpu().numpy().view(np.float64), np.sort(x))
    assert np.array_equal(res.origin.cpu().numpy(), ref.origin)
    y = rng.integers(-2**62, 2**62, p * npe, dtype=np.int64)
    res = run_gpu(y, [npe] * p, (16,), "deterministic", 3, "i", kind="i64")
    assert np.array_equal(res.keys.cpu().numpy(), np.sort(y))


def test_rlm_dropin_elements():
    """rlm_sort(net, data, plan, scheme, seed) returns the caller's own
    Element objects in the reference's order (tests/golden tiny cases)."""
    from paper_1410_6754_b200 import Element, LevelPlan, SeedSpec, rlm_sort

    class Net:
        p = 8

    g = RG.CASES["tiny_ragged"]
    data = {pe: [Element(k, pe, i) for i, k in enumerate(g["data"][str(pe)])] for pe in range(8)}
    out, reports = rlm_sort(Net(), data, LevelPlan(8, (2, 4)), "simple", SeedSpec(g["master_seed"], g["stream"]))
    offs = np.concatenate([[0], np.cumsum(g["input_pe_sizes"])])
    flat = [[int(e.key), int(offs[e.origin_pe]) + e.origin_pos] for pe in range(8) for e in out[pe]]
    assert flat == g["output"]
    assert [len(out[pe]) for pe in range(8)] == g["pe_sizes"]
    assert reports == g["reports"]
    ids = {id(e) for seq in data.values() for e in seq}
    assert all(id(e) in ids for seq in out.values() for e in seq)
    with pytest.raises(ValueError):
        rlm_sort(Net(), data, LevelPlan(4, (4,)), "simple", SeedSpec(0, "x"))


def test_rlm_large_balanced():
    """2^24 uniform u64, p=64 (8,8): output == numpy.sort, every PE exactly n/p."""
    n, p = 1 << 24, 64
    keys = np.random.default_rng(1).integers(0, 2**64, n, dtype=np.uint64)
    res = run_gpu(keys, [n // p] * p, (8, 8), "simple", 1, "algo/rep0")
    assert np.array_equal(res.keys.cpu().numpy().view(np.uint64), np.sort(keys))
    assert set(int(x) for x in res.pe_sizes) == {n // p}
    o = res.origin.cpu().numpy()
    assert np.array_equal(keys[o], np.sort(keys))


def test_rlm_payloads_and_ragged_sizes():
    """Payloads follow their keys; PEs of very different sizes (and empty
    ones) still end perfectly balanced (rlm.py:1-9)."""
    from oracle import rlm_oracle as R
    rng = np.random.default_rng(9)
    p = 16
    sizes = [0, 5000, 1, 0, 12000, 300, 300, 0, 7000, 2, 2, 2, 9000, 0, 0, 4096]
    n = sum(sizes)
    keys = rng.integers(0, 50, n, dtype=np.uint64)          # heavy duplicates: ties by origin
    vals = rng.integers(0, 2**62, n, dtype=np.int64)
    for scheme in ("simple", "randomized"):
        ref = R.rlm_sort(keys, sizes, (4, 4), scheme, 2, "r", vals=vals)
        res = run_gpu(keys, sizes, (4, 4), scheme, 2, "r", vals=vals)
        assert np.array_equal(res.keys.cpu().numpy().view(np.uint64), ref.keys)
        assert np.array_equal(res.origin.cpu().numpy(), ref.origin)
        assert np.array_equal(res.vals.cpu().numpy(), ref.vals)
        assert [int(x) for x in res.pe_sizes] == list(ref.pe_sizes)
        assert max(res.pe_sizes) - min(res.pe_sizes) <= 2
