"""Full-size parity on the B200 (BASELINE configs 2-5 at their own sizes).

The device run (one-call driver, reference-seeded sample streams) is compared
level by level with the full-size CPU oracle (oracle/fullsize.py, pinned to
the reference's fixtures and to oracle/ams_oracle.py in test_oracle.py):

* every group's sample size, bucket count, per-member bucket histogram,
  plan boundaries and loads (SURVEY §8 layout contract steps 1-4; ams.py:
  224-258), and the next level's member sizes (delivery.py:78-80);
* the final per-PE sizes and the whole output, bit for bit (the oracle's
  per-PE stable sorts, == numpy.sort);
* with payloads (config 5): payload == payload[argsort(keys, stable)] (F1).

Inputs follow BASELINE.json / SURVEY §8(d) exactly (seeded numpy
generators, host-made), not device stand-ins.  Each case costs one oracle
run on the GPU box's host cores (~1-2 min at 2^30).
"""

import gc

import numpy as np
import pytest
import torch

from oracle import ams_oracle as O
from oracle import fullsize as F

pytestmark = pytest.mark.gpu


def _sort_on_gpu(keys_np, p, groups, seed, kind, vals=False):
    from paper_1410_6754_b200 import AmsParams, SeedSpec, ams_sort_tensors
    n = len(keys_np)
    host = torch.from_numpy(keys_np.view(np.int64) if keys_np.dtype == np.uint64 else keys_np)
    d_keys = host.cuda()
    d_vals = torch.arange(n, dtype=torch.int64, device="cuda") if vals else None
    res = ams_sort_tensors(d_keys, [n // p] * p, AmsParams(tuple(groups), None, 16, 0.1),
                           SeedSpec(seed, "algo/rep0"), vals=d_vals, key_kind=kind)
    torch.cuda.synchronize()
    out = res.keys.cpu().numpy()
    ov = res.vals.cpu().numpy() if vals else None
    levels = res.levels
    sizes = [int(x) for x in res.pe_sizes]
    reports = res.reports
    del res, d_keys, d_vals
    torch.cuda.empty_cache()
    return out, ov, sizes, levels, reports


def _check(keys_np, p, groups, seed, kind="u64", vals=False, eps=0.1, bound=True):
    ordered = O.f64_to_ordered_u64(keys_np) if kind == "f64" else keys_np
    out, ov, sizes, levels, reports = _sort_on_gpu(keys_np, p, groups, seed, kind, vals)
    ref = F.ams_sort_fullsize(ordered, [len(keys_np) // p] * p, tuple(groups), None, 16, eps,
                              seed, "algo/rep0")
    bad = F.compare_levels(levels, ref)
    assert not bad, bad[:10]
    assert sizes == list(ref.pe_sizes)
    got = O.f64_to_ordered_u64(out.view(np.float64)) if kind == "f64" else out.view(np.uint64)
    assert np.array_equal(got, ref.keys), "output differs from the oracle"
    assert bool(np.all(got[1:] >= got[:-1]))
    if bound:  # the reference met its budget at these sizes
        assert max(sizes) <= (1 + eps) * len(keys_np) / p
        assert sum(r["over_budget"] for r in reports) == 0
    if vals:
        order = np.argsort(ordered, kind="stable")
        assert np.array_equal(ov, order), "payload is not the stable argsort"
    del out, ov, ref, got
    gc.collect()


def test_config2_full_size_oracle_levels():
    """Config 2 exactly: n=2^28 uint64 default_rng(1), p=64, (8,8)."""
    n = 1 << 28
    _check(np.random.default_rng(1).integers(0, 2**64, n, dtype=np.uint64), 64, (8, 8), 1)


@pytest.mark.parametrize("dist", ["zipf", "sorted", "reverse", "equal"])
def test_config2_shape_skewed_oracle_levels(dist):
    n = 1 << 28
    keys = {"zipf": lambda: O.zipf_keys(n, 4), "sorted": lambda: np.arange(n, dtype=np.uint64),
            "reverse": lambda: (n - 1 - np.arange(n)).astype(np.uint64),
            "equal": lambda: np.full(n, 42, np.uint64)}[dist]()
    _check(keys, 64, (8, 8), 1)


def test_config3_full_size_oracle_levels():
    """Config 3 on one GPU: n=2^30 float64 default_rng(2).random, p=256, (8,32)."""
    _check(np.random.default_rng(2).random(1 << 30), 256, (8, 32), 2, kind="f64")


@pytest.mark.parametrize("dist", ["zipf", "sorted", "reverse", "equal"])
def test_config4_full_size_oracle_levels(dist):
    """Config 4 on one GPU: n=2^30 uint64, p=256, (8,32): (a) Zipf(1.1) over
    2^10 values (default_rng(4)), (b) sorted, (c) reverse, (d) all 42."""
    n = 1 << 30
    keys = {"zipf": lambda: O.zipf_keys(n, 4), "sorted": lambda: np.arange(n, dtype=np.uint64),
            "reverse": lambda: (n - 1 - np.arange(n)).astype(np.uint64),
            "equal": lambda: np.full(n, 42, np.uint64)}[dist]()
    _check(keys, 256, (8, 32), 4)


@pytest.mark.parametrize("groups", [(256,), (8, 32)], ids=["k1", "k2"])
@pytest.mark.parametrize("log2n", [10, 12, 13, 14, 16, 18, 20, 22, 24, 27])
def test_config5_kv_oracle_levels(groups, log2n):
    """Config 5: uint64 keys with the origin index as payload, uniform
    default_rng(3), p=256, k=1 (256,) — 4096 buckets, the serial-rank
    scatter — and k=2 (8,32).  n covers the bench's one-GPU weak-scaling
    points (n = n/GPU = 2^10..2^24) and the whole 8-GPU problem (n = 8 n/GPU,
    SURVEY Appendix A: 2^13..2^27)."""
    n = 1 << log2n
    _check(np.random.default_rng(3).integers(0, 2**64, n, dtype=np.uint64), 256, groups, 3,
           vals=True, bound=log2n >= 17)


@pytest.mark.parametrize("groups", [(256,), (8, 32)], ids=["k1", "k2"])
def test_config5_keys_only_oracle_levels(groups):
    """Config 5's largest point keys-only (the bucket-major last level)."""
    n = 8 << 24
    _check(np.random.default_rng(3).integers(0, 2**64, n, dtype=np.uint64), 256, groups, 3)
