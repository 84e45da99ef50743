"""One cfg2-shaped sort for profiling (ncu); no timing printed.

    python tools/profile_case.py [log2n] [steps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6754_b200 import AmsParams, SeedSpec  # noqa: E402
from paper_1410_6754_b200.api import get_sorter  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n = 1 << log2n
keys = torch.from_numpy(np.random.default_rng(1).integers(0, 2**64, n, dtype=np.uint64).view(np.int64)).cuda()
s = get_sorter(0)
for _ in range(steps):
    res = s.sort(keys, [n // 64] * 64, AmsParams((8, 8), None, 16, 0.1), SeedSpec(1, "algo/rep0"),
                 key_kind="u64", with_stats=False)
torch.cuda.synchronize()
o = res.keys.view(torch.int64) ^ (-(2**63))
assert bool((o[1:] >= o[:-1]).all())
print("ok", res.launches)
