"""Time the CTA-local cell sort alone: n uniform keys split into segments of
`seg` keys (all <= the shared-memory capacity, so ams_final_sort sorts each
segment directly with k_smem_sort).  Checks the result.

    python tools/sortbench.py [log2n] [seg] [reps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6754_b200 import _lib as L  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
seg = int(sys.argv[2]) if len(sys.argv) > 2 else 6400
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
n = 1 << log2n
torch.cuda.set_device(0)
ctx = L.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
g = torch.Generator(device="cuda").manual_seed(1)
keys = torch.randint(-(2**63), 2**63 - 1, (n,), dtype=torch.int64, device="cuda", generator=g)
src = torch.empty_like(keys)
tmp = torch.empty_like(keys)
out = torch.empty_like(keys)
nseg = (n + seg - 1) // seg
sizes = np.full(nseg, seg, np.uint64)
sizes[-1] = n - seg * (nseg - 1)
offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.uint64)
ctx.set_timing(True)
for r in range(reps + 1):
    src.copy_(keys)
    if r == 1:
        ctx.reset_stats()
    ctx.final_sort(src, None, tmp, None, out, None, L.KEY_U64, offs, sizes)
torch.cuda.synchronize()
st = ctx.kernel_stats()
ms, by, la = st["smem_sort"]
o = out.view(torch.int64) ^ (-(2**63))
ok = True
for s0, c in [(int(offs[i]), int(sizes[i])) for i in (0, nseg // 2, nseg - 1)]:
    seg_o = o[s0:s0 + c]
    ok &= bool((seg_o[1:] >= seg_o[:-1]).all())
print(f"smem_sort n=2^{log2n} seg={seg}: {ms / reps:.3f} ms/rep  {by / (ms / 1e3) / 1e9:.0f} GB/s  "
      f"launches/rep {la / reps:.1f}  sorted={ok}  fallback/overflow={ctx.final_sort_stats()}")
