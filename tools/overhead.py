"""Per-sort overhead at small n (GPU work negligible): wall time of the public
tensor API and of the one-call C ABI, cfg2 parameters.
    python tools/overhead.py [log2n] [reps]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6754_b200 import AmsParams, SeedSpec  # noqa: E402
from paper_1410_6754_b200.api import get_sorter  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
n = 1 << log2n
keys = torch.from_numpy(np.random.default_rng(1).integers(0, 2**64, n, dtype=np.uint64).view(np.int64)).cuda()
out = torch.empty_like(keys)
s = get_sorter(0)
p = AmsParams((8, 8), None, 16, 0.1)
sizes = [n // 64] * 64
for ws in (False, True):
    run = lambda: s.sort(keys, sizes, p, SeedSpec(1, "algo/rep0"), out=out, key_kind="u64", with_stats=ws)
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) / reps * 1e3
    print(f"n=2^{log2n} with_stats={ws}: {e0.elapsed_time(e1) / reps:.3f} ms/sort (events), {wall:.3f} ms wall")
