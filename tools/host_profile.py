"""Wall-clock cost of each host-side step of one sort (small n: GPU time is
negligible, so this is the host overhead per sort).

    python tools/host_profile.py [log2n] [reps]
"""
import collections
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6754_b200 import AmsParams, SeedSpec, _lib as L  # noqa: E402
from paper_1410_6754_b200.api import get_sorter  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
n = 1 << log2n
acc = collections.defaultdict(float)


def wrap(obj, name):
    f = getattr(obj, name)

    def g(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        acc[name] += time.perf_counter() - t
        return r
    setattr(obj, name, g)


s = get_sorter(0)
for nm in ("level_sample", "level_splitters", "level_classify", "level_scatter", "final_sort",
           "set_stream"):
    wrap(s.ctx, nm)
for nm in ("draw_sample_positions", "plan_level"):
    wrap(L, nm)
keys = torch.from_numpy(np.random.default_rng(1).integers(0, 2**64, n, dtype=np.uint64).view(np.int64)).cuda()
p = AmsParams((8, 8), None, 16, 0.1)
for _ in range(3):
    s.sort(keys, [n // 64] * 64, p, SeedSpec(1, "algo/rep0"), key_kind="u64", with_stats=False)
torch.cuda.synchronize()
acc.clear()
t0 = time.perf_counter()
for _ in range(reps):
    s.sort(keys, [n // 64] * 64, p, SeedSpec(1, "algo/rep0"), key_kind="u64", with_stats=False)
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / reps
print(f"n=2^{log2n}: {tot * 1e3:.3f} ms per sort (wall)")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:24s} {v / reps * 1e3:8.3f} ms")
print(f"  {'(python rest)':24s} {(tot - sum(acc.values()) / reps) * 1e3:8.3f} ms")
