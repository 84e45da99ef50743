"""Small sorts through every device path (fixed cells, exact cells, KV
rounds, delivery schemes, overflow fallback), each checked against numpy.sort:
    python tools/paths_case.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6754_b200 import AmsParams, SeedSpec  # noqa: E402
from paper_1410_6754_b200.api import get_sorter  # noqa: E402

s = get_sorter(0)
rng = np.random.default_rng(0)
for groups, b, npe, vals, scheme, dist in [
        ((4,), 4, 1 << 15, False, "simple", "uniform"),       # fixed-capacity final path
        ((2, 4), 4, 1 << 14 | 7, False, "simple", "dense"),     # odd sizes, exact cells
        ((2, 4), 4, 1 << 14, True, "simple", "uniform"),        # KV: exact digit rounds
        ((4, 4), 8, 3001, True, "deterministic", "few"),        # tags + relayout
        ((4, 4), 8, 3001, False, "randomized", "uniform"),
        ((8,), 4, 20000, False, "simple", "clustered"),         # overflow fallback
        ((256,), 16, 300, True, "simple", "uniform"),           # 4096 buckets: serial stable ranks
        ((256,), 16, 300, False, "simple", "uniform"),          # 4096 buckets, bucket-major keys-only
        ((2, 32), 16, 2000, True, "simple", "uniform"),         # 512 buckets: 16-bit stored ids
        ((2, 2), 4, 0, False, "simple", "uniform")]:            # empty input
    p = int(np.prod(groups))
    n = p * npe
    if dist == "uniform":
        keys = rng.integers(0, 2**64, n, dtype=np.uint64)
    elif dist == "dense":
        keys = np.arange(n, dtype=np.uint64)[::-1].copy()
    elif dist == "few":
        keys = rng.integers(0, 5, n).astype(np.uint64)
    else:
        c = rng.integers(0, 2**60, 3, dtype=np.uint64)
        keys = c[rng.integers(0, 3, n)] + rng.integers(0, 1 << 14, n).astype(np.uint64)
    d = torch.from_numpy(keys.view(np.int64)).cuda()
    v = torch.arange(n, dtype=torch.int64, device="cuda") if vals else None
    res = s.sort(d, [npe] * p, AmsParams(groups, None, b, 0.1), SeedSpec(3, "algo/rep0"), vals=v,
                 key_kind="u64", with_stats=False, scheme=scheme)
    torch.cuda.synchronize()
    out = res.keys.cpu().numpy().view(np.uint64)
    assert np.array_equal(out, np.sort(keys)), (groups, dist)
    print("ok", groups, scheme, dist, "vals" if vals else "keys")
