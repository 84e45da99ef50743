"""Device timeline of one cfg2 sort: every timed launch with its start/end
and the idle gap before it (host round trips show up as gaps).

    python tools/timeline.py [log2n]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6754_b200 import AmsParams, SeedSpec  # noqa: E402
from paper_1410_6754_b200.api import get_sorter  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
n = 1 << log2n
keys = torch.from_numpy(np.random.default_rng(1).integers(0, 2**64, n, dtype=np.uint64).view(np.int64)).cuda()
s = get_sorter(0)
p = AmsParams((8, 8), None, 16, 0.1)
run = lambda: s.sort(keys, [n // 64] * 64, p, SeedSpec(1, "algo/rep0"), key_kind="u64", with_stats=False)
for _ in range(3):
    run()
torch.cuda.synchronize()
s.ctx.set_timing(True)
s.ctx.reset_stats()
run()
run()
torch.cuda.synchronize()
tl = s.ctx.timeline()
s.ctx.set_timing(False)
prev = None
busy = gaps = 0.0
# the second sort only (the first one warms the event pool)
half = len(tl) // 2
t_first = tl[half][1]
for name, t0, t1 in tl[half:]:
    gap = 0.0 if prev is None else t0 - prev
    gaps += max(gap, 0.0)
    busy += t1 - t0
    print(f"{t0 - t_first:9.3f} {t1 - t0:8.3f}  gap {gap:7.3f}  {name}")
    prev = t1
print(f"busy {busy:.3f} ms, gaps {gaps:.3f} ms, span {prev - t_first:.3f} ms")
