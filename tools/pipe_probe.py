import sys, os, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6754_b200 import AmsParams, SeedSpec
from paper_1410_6754_b200.api import HostSortPipeline
n = 1 << 28
keys = torch.from_numpy(np.random.default_rng(1).integers(0, 2**64, n, dtype=np.uint64).view(np.int64))
h_in = keys.pin_memory(); h_out = torch.empty_like(h_in).pin_memory()
pipe = HostSortPipeline(n, [n // 64] * 64, AmsParams((8, 8), None, 16, 0.1), SeedSpec(1, "algo/rep0"))
pipe.run([h_in], [h_out]); torch.cuda.synchronize()
for K in (1, 2, 4, 6):
    t = time.perf_counter(); pipe.run([h_in] * K, [h_out] * K); torch.cuda.synchronize()
    print(K, f"{(time.perf_counter() - t) * 1e3 / K:.1f} ms/step")
# host time inside sort
s = pipe.sorter
t = time.perf_counter(); s.sort(pipe.d_in[0][:n], [n // 64] * 64, pipe.params, pipe.seed, out=pipe.d_out[0][:n], key_kind="u64", with_stats=False); t1 = time.perf_counter(); torch.cuda.synchronize()
print("sort call returns after", (t1 - t) * 1e3, "ms; done after", (time.perf_counter() - t) * 1e3)
