"""HostSortPipeline period with and without the sort (copies only), cfg2."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6754_b200 import AmsParams, SeedSpec
from paper_1410_6754_b200.api import HostSortPipeline
n = 1 << 28
sizes = [n // 64] * 64
pipe = HostSortPipeline(n, sizes, AmsParams((8, 8), None, 16, 0.1), SeedSpec(1, "algo/rep0"))
ins = [torch.from_numpy(np.random.default_rng(i).integers(0, 2**63, n, dtype=np.int64)).pin_memory() for i in range(2)]
outs = [torch.empty(n, dtype=torch.int64).pin_memory() for _ in range(2)]
K = 8
for mode in ("sort", "copy-only"):
    if mode == "copy-only":
        class Fake:
            def sort(self, x, *a, out=None, **k):
                out.copy_(x)
                class R: pe_sizes = None
                return R()
        pipe.sorter = Fake()
    ev = []
    pipe.run([ins[i % 2] for i in range(K)], [outs[i % 2] for i in range(K)], done_events=ev)
    torch.cuda.synchronize()
    gaps = [ev[i].elapsed_time(ev[i + 1]) for i in range(len(ev) - 1)]
    print(mode, "period ms:", " ".join(f"{g:.1f}" for g in gaps))
