"""Device timeline of one sort of any shape: every timed launch with its
start/end and the idle gap before it (host round trips show up as gaps).

    python tools/timeline_case.py LOG2N P GROUPS [kv] [a]
    e.g. tools/timeline_case.py 20 16 16 0 16     (config 1)
         tools/timeline_case.py 12 256 256 1      (config 5, k=1)
         tools/timeline_case.py 24 256 8,32 1     (config 5, k=2)
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6754_b200 import AmsParams, SeedSpec  # noqa: E402
from paper_1410_6754_b200.api import get_sorter  # noqa: E402

log2n, p = int(sys.argv[1]), int(sys.argv[2])
groups = tuple(int(x) for x in sys.argv[3].split(","))
kv = len(sys.argv) > 4 and sys.argv[4] == "1"
a = float(sys.argv[5]) if len(sys.argv) > 5 else None
n = 1 << log2n
keys = torch.from_numpy(np.random.default_rng(3).integers(0, 2**64, n, dtype=np.uint64).view(np.int64)).cuda()
vals = torch.arange(n, dtype=torch.int64, device="cuda") if kv else None
ok_, ov_ = torch.empty_like(keys), (torch.empty_like(vals) if kv else None)
s = get_sorter(0)
prm = AmsParams(groups, a, 16, 0.1)
run = lambda: s.sort(keys, [n // p] * p, prm, SeedSpec(3, "algo/rep0"), vals=vals, out=ok_, out_vals=ov_,
                     key_kind="u64", with_stats=False)
for _ in range(3):
    run()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    run()
t_host = (time.perf_counter() - t) / 10
torch.cuda.synchronize()
t_all = (time.perf_counter() - t) / 10
s.ctx.set_timing(True)
s.ctx.reset_stats()
run()
run()
torch.cuda.synchronize()
tl = s.ctx.timeline()
s.ctx.set_timing(False)
prev = None
busy = gaps = 0.0
half = len(tl) // 2
t_first = tl[half][1]
print(f"== n=2^{log2n} p={p} groups={groups} kv={kv}: host call {1e3 * t_host:.3f} ms, "
      f"back-to-back {1e3 * t_all:.3f} ms per sort")
for name, t0, t1 in tl[half:]:
    gap = 0.0 if prev is None else t0 - prev
    gaps += max(gap, 0.0)
    busy += t1 - t0
    print(f"{t0 - t_first:9.3f} {t1 - t0:8.3f}  gap {gap:7.3f}  {name}")
    prev = t1
print(f"busy {busy:.3f} ms, gaps {gaps:.3f} ms, span {prev - t_first:.3f} ms")
