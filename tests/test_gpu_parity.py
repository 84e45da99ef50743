"""GPU parity: the CUDA path (through libams_b200.so) against the reference's
golden fixtures and the CPU oracle.

Bar: output bit-exact with the reference and numpy.sort;
per-level splitters, histograms, plans and member sizes identical to the
reference when the sample streams are the same; per-PE sizes within
(1+eps)·n/p where the reference met its budget; stable payload order.
"""

import re

import numpy as np
import pytest
import torch

from oracle import ams_oracle as O
from tests import golden_util as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_1410_6754_b200 import api as A
    return A


def dev_u64(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).cuda()


def host_u64(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


def run_gpu(api, keys, sizes, groups, a, b, eps, master, stream, vals=True, record=True,
            scheme="simple"):
    from paper_1410_6754_b200 import AmsParams, SeedSpec
    d_keys = dev_u64(keys)
    d_vals = torch.arange(len(keys), dtype=torch.int64, device="cuda") if vals else None
    res = api.ams_sort_tensors(d_keys, sizes, AmsParams(tuple(groups), a, b, eps),
                               SeedSpec(master, stream), vals=d_vals, key_kind="u64",
                               record_splitters=record, scheme=scheme)
    torch.cuda.synchronize()
    return res


def check_levels(res, g):
    assert len(res.levels) == len(g["levels"])
    for lv, (rec, refs) in enumerate(zip(res.levels, g["levels"])):
        assert len(rec.group_first) == len(refs)
        row = 0
        for gi, ref in enumerate(refs):
            P = int(rec.group_npe[gi])
            assert int(rec.sample_size[gi]) == ref["sample_size"]
            assert int(rec.bucket_count[gi]) == ref["bucket_count"]
            nb = ref["bucket_count"]
            ghist = rec.seg_hist[row:row + P, :nb].astype(np.int64).sum(axis=0)
            assert ghist.tolist() == ref["global_hist"], f"level {lv} group {gi} histogram"
            assert [int(x) for x in rec.boundaries[gi]] == ref["boundaries"]
            assert [int(x) for x in rec.loads[gi]] == ref["loads"]
            assert [int(x) for x in rec.new_sizes[row:row + P]] == ref["new_sizes"]
            if rec.splitters:
                sk, sp = rec.splitters[gi]
                assert [int(x) for x in sk] == ref["splitter_keys"], f"level {lv} group {gi} splitters"
                assert [int(x) for x in sp] == ref["splitter_pos"]
            row += P
    for mine, ref in zip(res.reports, g["reports"]):
        for k, v in ref.items():
            assert mine[k] == v, (k, mine[k], v)


NON_SIMPLE = ("det_", "perm_", "rand_")  # fixtures of the other delivery schemes


@pytest.mark.parametrize("name,native",
                         [(n, True) for n in G.names()]
                         + [(n, False) for n in G.names() if not n.startswith(NON_SIMPLE)],
                         ids=lambda v: {True: "c_driver", False: "py_levels"}.get(v, v)
                         if isinstance(v, bool) else v)
def test_golden_parity(api, name, native):
    """Both host drivers: the one-call C++ ams_sort_run (native) and, for
    scheme="simple", the Python level loop over the level entry points
    (which also reads the splitters back for comparison)."""
    g = G.load(name)
    scheme = g.get("scheme", "simple")
    keys, sizes = G.input_of(g)
    if "error" in g:  # the reference rejects this input: same exception class and message
        exc = {"ValueError": ValueError, "RuntimeError": RuntimeError}[g["error"]["type"]]
        with pytest.raises(exc, match=re.escape(g["error"]["message"])):
            run_gpu(api, keys, sizes, g["groups"], g["a"], g["b"], g["eps"], g["master_seed"],
                    g["stream"], record=False, scheme=scheme)
        return
    assert G.sha_u64(keys) == g["input_sha256"]
    res = run_gpu(api, keys, sizes, g["groups"], g["a"], g["b"], g["eps"], g["master_seed"],
                  g["stream"], record=not native, scheme=scheme)
    out = host_u64(res.keys)
    assert [int(x) for x in res.pe_sizes] == g["pe_sizes"]
    assert G.sha_u64(out) == g["output_sha256"]
    assert G.sha_i64(res.vals.cpu().numpy()) == g["origin_sha256"]
    check_levels(res, g)


@pytest.mark.parametrize("scheme", ["deterministic", "permuted", "randomized"])
def test_per_level_driver_rejects_other_schemes(api, scheme):
    """record_splitters runs the per-level host driver, which implements the
    simple scheme only: the other schemes fail loudly instead of silently
    delivering with simple's placement."""
    keys = np.arange(64, dtype=np.uint64)[::-1].copy()
    with pytest.raises(ValueError, match="simple scheme only"):
        run_gpu(api, keys, [8] * 8, [8], None, 16, 0.1, 1, "s", record=True, scheme=scheme)


@pytest.mark.parametrize("name", [n for n in G.names()
                                  if n.startswith(("tiny", "det_tiny", "perm_tiny", "rand_tiny"))])
def test_dropin_elements(api, name):
    """ams_sort(net, data, params, scheme, seed) returns the reference's
    exact per-PE Element lists."""
    from paper_1410_6754_b200 import AmsParams, Element, SeedSpec

    class Net:
        def __init__(self, p):
            self.p = p

    g = G.load(name)
    p = g["p"]
    data = {pe: [Element(k, o, i) for k, o, i in g["data"][str(pe)]] for pe in range(p)}
    call = lambda: api.ams_sort(Net(p), data, AmsParams(tuple(g["groups"]), g["a"], g["b"], g["eps"]),
                                g.get("scheme", "simple"), SeedSpec(g["master_seed"], g["stream"]))
    if "error" in g:
        with pytest.raises(ValueError, match=re.escape(g["error"]["message"])):
            call()
        return
    out, reports = call()
    flat = [list(e) for pe in range(p) for e in out[pe]]
    assert flat == g["output"]
    assert [len(out[pe]) for pe in range(p)] == g["pe_sizes"]
    for mine, ref in zip(reports, g["reports"]):
        for k, v in ref.items():
            assert mine[k] == v


@pytest.mark.parametrize("groups,npe,dist", [
    ((8, 8), 1 << 12, "uniform"), ((8, 8), 3000, "zipf"), ((4, 4, 4), 2048, "uniform"),
    ((8, 32), 1 << 10, "sorted"), ((8, 32), 1 << 10, "reverse"), ((8, 32), 1 << 10, "equal"),
    ((16,), 1 << 16, "uniform"), ((2, 8), 50_000, "few"), ((64,), 777, "uniform"),
    ((256,), 64, "uniform"), ((8, 32), 4096, "zipf"),
])
@pytest.mark.parametrize("native", [True, False], ids=["c_driver", "py_levels"])
def test_oracle_parity_random(api, groups, npe, dist, native):
    """Seeded inputs beyond the fixtures, checked level by level against the
    oracle (itself pinned to the reference)."""
    p = int(np.prod(groups))
    n = p * npe
    rng = np.random.default_rng(hash((groups, npe, dist)) & 0xFFFF)
    if dist == "uniform":
        keys = rng.integers(0, 2**64, n, dtype=np.uint64)
    elif dist == "zipf":
        keys = O.zipf_keys(n, 11)
    elif dist == "sorted":
        keys = np.arange(n, dtype=np.uint64)
    elif dist == "reverse":
        keys = (n - 1 - np.arange(n)).astype(np.uint64)
    elif dist == "equal":
        keys = np.full(n, 42, dtype=np.uint64)
    else:  # few distinct values spread over the whole range
        keys = rng.choice(np.array([0, 1, 2**40, 2**63, 2**64 - 1], dtype=np.uint64), n)
    sizes = [npe] * p
    vals = np.arange(n, dtype=np.int64)
    ref = O.ams_sort(keys, sizes, groups, None, 16, 0.1, 77, "algo/rep0", vals=vals)
    res = run_gpu(api, keys, sizes, groups, None, 16, 0.1, 77, "algo/rep0", record=not native)
    out = host_u64(res.keys)
    assert np.array_equal(out, ref.keys)
    assert np.array_equal(res.vals.cpu().numpy(), ref.vals)
    assert [int(x) for x in res.pe_sizes] == list(ref.pe_sizes)
    for rec, infos in zip(res.levels, ref.levels):
        for gi, info in enumerate(infos):
            assert [int(x) for x in rec.boundaries[gi]] == list(info.plan.boundaries)
            if not native:
                sk, sp = rec.splitters[gi]
                assert np.array_equal(sk, info.splitter_keys)
                assert np.array_equal(sp.astype(np.int64), info.splitter_pos)
    for mine, theirs in zip(res.reports, ref.reports):
        for k, v in theirs.items():
            assert mine[k] == v, (k, mine[k], v)


@pytest.mark.parametrize("groups,npe,dist", [
    ((8, 8), 1 << 12, "equal"), ((8, 8), 1 << 12, "sorted"), ((8, 8), 3000, "zipf"),
    ((4, 4, 4), 1024, "few"), ((8, 32), 1 << 9, "equal"), ((2, 8), 5000, "uniform"),
])
@pytest.mark.parametrize("with_vals", [True, False], ids=["kv", "keys"])
@pytest.mark.parametrize("scheme", ["deterministic", "permuted", "randomized"])
def test_oracle_parity_deterministic(api, groups, npe, dist, with_vals, scheme):
    """scheme="deterministic" (delivery.py:188-306: two-phase assignment)
    and "permuted" (delivery.py:183-185: Feistel enumeration): member
    placement differs from "simple", ties broken by the carried origin tags."""
    p = int(np.prod(groups))
    n = p * npe
    rng = np.random.default_rng(hash((groups, npe, dist, 7)) & 0xFFFF)
    if dist == "uniform":
        keys = rng.integers(0, 2**64, n, dtype=np.uint64)
    elif dist == "zipf":
        keys = O.zipf_keys(n, 13)
    elif dist == "sorted":
        keys = np.arange(n, dtype=np.uint64)
    elif dist == "equal":
        keys = np.full(n, 42, dtype=np.uint64)
    else:
        keys = rng.choice(np.array([0, 1, 2**40, 2**63, 2**64 - 1], dtype=np.uint64), n)
    sizes = [npe] * p
    vals = np.arange(n, dtype=np.int64)
    ref = O.ams_sort(keys, sizes, groups, None, 16, 0.1, 78, "algo/rep0", vals=vals, scheme=scheme)
    res = run_gpu(api, keys, sizes, groups, None, 16, 0.1, 78, "algo/rep0", vals=with_vals,
                  record=False, scheme=scheme)
    assert np.array_equal(host_u64(res.keys), ref.keys)
    if with_vals:
        assert np.array_equal(res.vals.cpu().numpy(), ref.vals)
    assert [int(x) for x in res.pe_sizes] == list(ref.pe_sizes)
    for rec, infos in zip(res.levels, ref.levels):
        row = 0
        for gi, info in enumerate(infos):
            assert [int(x) for x in rec.boundaries[gi]] == list(info.plan.boundaries)
            P = len(info.new_sizes)
            assert [int(x) for x in rec.new_sizes[row:row + P]] == list(info.new_sizes)
            row += P
    for mine, theirs in zip(res.reports, ref.reports):
        for k, v in theirs.items():
            assert mine[k] == v, (k, mine[k], v)


@pytest.mark.parametrize("groups,b,npe,dist", [
    ((4,), 4, 1 << 18, "uniform"), ((2, 4), 4, 1 << 18, "zipf"), ((4,), 4, 300_001, "equal"),
    ((2, 2, 2), 2, 1 << 18, "few"), ((2, 4), 4, 1 << 18, "sorted"), ((4,), 4, 199_999, "reverse"),
    ((16,), 16, 1 << 16, "uniform"), ((4,), 4, 1 << 18, "f64"), ((2, 2), 4, 1 << 19, "narrow"),
    ((4,), 4, 1 << 18, "clustered"), ((8, 8), 16, 1 << 12, "uniform"),
])
@pytest.mark.parametrize("with_stats,record", [(True, False), (False, False), (True, True)],
                         ids=["stats", "nostats", "py_levels"])
def test_oracle_parity_keys_only(api, groups, b, npe, dist, with_stats, record):
    """Keys-only sorts take the bucket-major last level and the
    fixed-capacity final partition (buckets above shared memory; counting-
    only cells for few-valued buckets, exact rounds for overflowed buckets):
    same output, per-PE sizes and plans as the oracle."""
    from paper_1410_6754_b200 import AmsParams, SeedSpec
    p = int(np.prod(groups))
    n = p * npe
    rng = np.random.default_rng(hash((groups, npe, dist, 3)) & 0xFFFF)
    if dist == "uniform":
        keys = rng.integers(0, 2**64, n, dtype=np.uint64)
    elif dist == "zipf":
        keys = O.zipf_keys(n, 12)
    elif dist == "equal":
        keys = np.full(n, 7, dtype=np.uint64)
    elif dist == "sorted":
        keys = np.arange(n, dtype=np.uint64)
    elif dist == "reverse":
        keys = (n - 1 - np.arange(n)).astype(np.uint64)
    elif dist == "f64":  # order-mapped doubles: density doubles across binade boundaries
        keys = O.f64_to_ordered_u64(rng.random(n))
    elif dist == "narrow":  # few distinct values per bucket: counting-only cells
        keys = rng.integers(1000, 1000 + 20_000, n).astype(np.uint64)
    elif dist == "clustered":  # dense clusters inside wide buckets: cells overflow
        centers = rng.integers(0, 2**60, 6, dtype=np.uint64)
        keys = centers[rng.integers(0, 6, n)] + rng.integers(0, 1 << 16, n).astype(np.uint64)
    else:
        keys = rng.choice(np.array([0, 1, 2**40, 2**63, 2**64 - 1], dtype=np.uint64), n)
    sizes = [npe] * p
    ref = O.ams_sort(keys, sizes, groups, None, b, 0.1, 79, "algo/rep0", with_stats=False)
    ctx = api.get_sorter(0).ctx
    before = ctx.final_sort_stats()
    res = api.get_sorter(0).sort(dev_u64(keys), sizes, AmsParams(tuple(groups), None, b, 0.1),
                                 SeedSpec(79, "algo/rep0"), key_kind="u64", with_stats=with_stats,
                                 record_splitters=record)
    torch.cuda.synchronize()
    after = ctx.final_sort_stats()
    if npe * p // (int(np.prod(groups)) * b) > 2 * 4096:  # buckets well above shared memory
        assert after["fixed_buckets"] > before["fixed_buckets"]  # the fixed-capacity path ran
    if dist == "clustered":  # and its exact fallback
        assert after["fixed_overflow_buckets"] > before["fixed_overflow_buckets"]
    if dist in ("uniform", "sorted", "reverse", "narrow", "equal"):
        # these never need the LSD fallback (dense ranges take the exact cell map)
        assert after["fallback_cells"] == before["fallback_cells"]
    assert np.array_equal(host_u64(res.keys), ref.keys)
    assert [int(x) for x in res.pe_sizes] == list(ref.pe_sizes)
    for rec, infos in zip(res.levels, ref.levels):
        for gi, info in enumerate(infos):
            assert [int(x) for x in rec.boundaries[gi]] == list(info.plan.boundaries)
        assert [int(x) for x in rec.new_sizes] == [s for info in infos for s in info.new_sizes]
    for mine, theirs in zip(res.reports, ref.reports):
        for k, v in theirs.items():
            assert mine[k] == v, (k, mine[k], v)


def test_ragged_and_empty_pes(api):
    rng = np.random.default_rng(5)
    sizes = [0, 5, 0, 0, 10_000, 1, 3, 0] + [int(x) for x in rng.integers(0, 3000, 56)]
    n = sum(sizes)
    keys = rng.integers(0, 1000, n).astype(np.uint64)
    ref = O.ams_sort(keys, sizes, (8, 8), None, 16, 0.2, 3, "root", vals=np.arange(n))
    res = run_gpu(api, keys, sizes, (8, 8), None, 16, 0.2, 3, "root")
    assert np.array_equal(host_u64(res.keys), ref.keys)
    assert np.array_equal(res.vals.cpu().numpy(), ref.vals)
    assert [int(x) for x in res.pe_sizes] == list(ref.pe_sizes)


def test_empty_input(api):
    res = run_gpu(api, np.zeros(0, np.uint64), [0] * 4, (2, 2), None, 16, 0.2, 1, "root")
    assert res.keys.numel() == 0 and list(res.pe_sizes) == [0] * 4


def test_float64_and_int64_keys(api):
    from paper_1410_6754_b200 import AmsParams, SeedSpec
    rng = np.random.default_rng(2)
    n = 1 << 20
    f = rng.standard_normal(n) * 1e3
    f[:10] = [0.0, 1.5, -1.5, np.inf, -np.inf, 1e-300, -1e-300, 3.0, 3.0, -2.0]
    res = api.ams_sort_tensors(torch.from_numpy(f).cuda(), [n // 16] * 16, AmsParams((4, 4)),
                               SeedSpec(1))
    assert np.array_equal(res.keys.cpu().numpy(), np.sort(f))
    i = rng.integers(-2**63, 2**63 - 1, n, dtype=np.int64)
    res = api.ams_sort_tensors(torch.from_numpy(i).cuda(), [n // 16] * 16, AmsParams((16,)),
                               SeedSpec(1))
    assert np.array_equal(res.keys.cpu().numpy(), np.sort(i))


def test_deterministic_repeat(api):
    rng = np.random.default_rng(9)
    n = 1 << 21
    keys = rng.integers(0, 2**64, n, dtype=np.uint64)
    a = run_gpu(api, keys, [n // 64] * 64, (8, 8), None, 16, 0.1, 1, "algo/rep0", record=False)
    ka, va = host_u64(a.keys).copy(), a.vals.cpu().numpy().copy()
    b = run_gpu(api, keys, [n // 64] * 64, (8, 8), None, 16, 0.1, 1, "algo/rep0", record=False)
    assert np.array_equal(ka, host_u64(b.keys)) and np.array_equal(va, b.vals.cpu().numpy())


def _wrap_checksums(t: torch.Tensor):
    """Multiset checksums of 64-bit patterns (wrapping int64 sums of x and x^2)."""
    x = t.view(torch.int64)
    return int(x.sum()), int((x * x).sum())


def _check_sorted_perm(inp: torch.Tensor, res, n: int, p: int, eps: float):
    out = res.keys
    assert out.numel() == n
    assert bool((out[1:] >= out[:-1]).all())
    assert _wrap_checksums(out) == _wrap_checksums(inp)
    assert int(np.asarray(res.pe_sizes).sum()) == n
    assert int(np.asarray(res.pe_sizes).max()) <= (1 + eps) * n / p


@pytest.mark.parametrize("scheme", ["deterministic", "permuted", "randomized"])
def test_config2_full_size_schemes(api, scheme):
    """Config 2 shape (n=2^28 uint64, p=64, (8,8)) at full size through the
    other delivery schemes, with origin payloads: sorted output, and the
    payload is the permutation that gathers the input into it."""
    from paper_1410_6754_b200 import AmsParams, SeedSpec
    n, p = 1 << 28, 64
    g = torch.Generator(device="cuda").manual_seed(1)
    keys = torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device="cuda", generator=g)
    vals = torch.arange(n, dtype=torch.int64, device="cuda")
    res = api.ams_sort_tensors(keys, [n // p] * p, AmsParams((8, 8), None, 16, 0.1),
                               SeedSpec(1, "algo/rep0"), vals=vals, key_kind="u64",
                               scheme=scheme)
    torch.cuda.synchronize()
    flip = torch.tensor(-(2**63), dtype=torch.int64, device="cuda")
    signed = res.keys.view(torch.int64) ^ flip  # unsigned order as signed order
    assert bool((signed[1:] >= signed[:-1]).all())
    assert torch.equal(keys[res.vals], res.keys.view(torch.int64))
    assert int(np.asarray(res.pe_sizes).sum()) == n
    del res, keys, vals, signed
    torch.cuda.empty_cache()


def test_host_pipeline_batches(api):
    """HostSortPipeline: several host batches with overlapped copies, each
    equal to the one-shot sort (and to numpy.sort)."""
    from paper_1410_6754_b200 import AmsParams, SeedSpec
    p, npe = 64, 5000
    n = p * npe
    rng = np.random.default_rng(5)
    batches = [rng.integers(0, 2**64, n, dtype=np.uint64) for _ in range(3)]
    ins = [torch.from_numpy(b.view(np.int64).copy()).pin_memory() for b in batches]
    outs = [torch.empty(n, dtype=torch.int64).pin_memory() for _ in batches]
    pipe = api.HostSortPipeline(n, [npe] * p, AmsParams((8, 8), None, 16, 0.1),
                                SeedSpec(1, "algo/rep0"))
    sizes = pipe.run(ins, outs)
    for b, o, sz in zip(batches, outs, sizes):
        assert np.array_equal(o.numpy().view(np.uint64), np.sort(b))
        ref = O.ams_sort(b, [npe] * p, (8, 8), None, 16, 0.1, 1, "algo/rep0")
        assert [int(x) for x in sz] == list(ref.pe_sizes)



@pytest.mark.gpu
@pytest.mark.parametrize("ndistinct", [1 << 14, 1 << 18])
def test_many_fallback_cells_keys_only(api, ndistinct):
    """Keys-only fast path with thousands of clustered cells (a few key
    values per cell, each repeated well above the cell sort's fix-up bound):
    the LSD fallback list is far longer than its speculative launch, so the
    deferred remainder launch runs too.  Output == numpy.sort."""
    from paper_1410_6754_b200 import AmsParams, SeedSpec
    from paper_1410_6754_b200.api import get_sorter
    n, p = 1 << 24, 64
    rng = np.random.default_rng(ndistinct)
    values = rng.integers(0, 2**64, ndistinct, dtype=np.uint64)
    keys = values[rng.integers(0, ndistinct, n)]
    d_keys = torch.from_numpy(keys.view(np.int64)).cuda()
    sorter = get_sorter(0)
    before = sorter.ctx.final_sort_stats()
    res = api.ams_sort_tensors(d_keys, [n // p] * p, AmsParams((8, 8), None, 16, 0.1), SeedSpec(3, "f"),
                               key_kind="u64")
    torch.cuda.synchronize()
    after = sorter.ctx.final_sort_stats()
    assert np.array_equal(res.keys.cpu().numpy().view(np.uint64), np.sort(keys))
    if ndistinct == 1 << 14:
        assert after["fallback_cells"] - before["fallback_cells"] > 256, \
            "expected more fallback cells than the speculative launch"


@pytest.mark.gpu
@pytest.mark.parametrize("groups,npe,dist,with_vals", [
    ((8, 8), 4096, "uniform", False), ((8, 8), 4096, "uniform", True), ((4, 4), 3000, "zipf", True),
    ((16,), 65536, "uniform", False), ((2, 2, 4), 700, "sorted", False), ((256,), 64, "uniform", True),
    ((4, 2), 5, "uniform", False),
])
def test_device_sample_mode(api, groups, npe, dist, with_vals):
    """sample_mode="device": stratified positions drawn on the
    GPU with the reference's quota split.  Bucket boundaries differ from the
    reference's, everything else holds: output == numpy.sort, payloads ==
    stable argsort, sample sizes as draw_sample's, the per-level load budget
    (ams.py:258) and determinism per seed."""
    from paper_1410_6754_b200 import AmsParams, SeedSpec
    p = int(np.prod(groups))
    n = p * npe
    rng = np.random.default_rng(p + npe)
    keys = {"uniform": lambda: rng.integers(0, 2**64, n, dtype=np.uint64),
            "zipf": lambda: O.zipf_keys(n, 11), "sorted": lambda: np.arange(n, dtype=np.uint64)}[dist]()
    d_keys = dev_u64(keys)
    d_vals = torch.arange(n, dtype=torch.int64, device="cuda") if with_vals else None
    prm = AmsParams(tuple(groups), None, 16, 0.2)
    runs = []
    for _ in range(2):
        res = api.ams_sort_tensors(d_keys, [npe] * p, prm, SeedSpec(7, "algo/rep0"), vals=d_vals,
                                   key_kind="u64", sample_mode="device")
        torch.cuda.synchronize()
        runs.append(res)
    res = runs[0]
    out = res.keys.cpu().numpy().view(np.uint64)
    assert np.array_equal(out, np.sort(keys))
    if with_vals:
        assert np.array_equal(res.vals.cpu().numpy(), np.argsort(keys, kind="stable"))
    assert int(np.sum(res.pe_sizes)) == n
    ref = O.ams_sort(keys, [npe] * p, groups, None, 16, 0.2, 7, "algo/rep0")
    for rec, infos in zip(res.levels, ref.levels):
        assert [int(x) for x in rec.sample_size] == [i.sample_size for i in infos]   # same quota split
    if dist == "uniform" and npe >= 64:
        assert max(int(x) for x in res.pe_sizes) <= 1.2 * n / p + 1
    assert [int(x) for x in runs[1].pe_sizes] == [int(x) for x in res.pe_sizes]      # deterministic per seed
    with pytest.raises(ValueError):
        api.ams_sort_tensors(d_keys, [npe] * p, prm, SeedSpec(7, "x"), key_kind="u64", sample_mode="device",
                             record_holders=True)
