"""Host-side step times of ams_sort_run (AMS_HOST_TRACE=1) for cfg2-shaped
sorts, next to the device time of the same sorts.
    AMS_HOST_TRACE=1 python tools/host_trace.py [log2n] [reps]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6754_b200 import AmsParams, SeedSpec  # noqa: E402
from paper_1410_6754_b200.api import get_sorter  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
n = 1 << log2n
keys = torch.from_numpy(np.random.default_rng(1).integers(0, 2**64, n, dtype=np.uint64).view(np.int64)).cuda()
out = torch.empty_like(keys)
s = get_sorter(0)
p = AmsParams((8, 8), None, 16, 0.1)
for i in range(reps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record()
    s.sort(keys, [n // 64] * 64, p, SeedSpec(1, "algo/rep0"), out=out, key_kind="u64", with_stats=False)
    t_ret = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    print(f"sort {i}: device {e0.elapsed_time(e1):.3f} ms, host call {1e3 * (t_ret - t):.3f} ms",
          file=sys.stderr, flush=True)
