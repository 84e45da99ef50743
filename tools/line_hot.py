"""Aggregate an ncu `--print-source cuda,sass` CSV by CUDA source line:
warp-instructions executed and stall samples per line."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(open(path)))
agg = defaultdict(lambda: [0, 0, ""])
fname = ""
hdr = None
cur_line = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    # cuda rows: Line No, Source, then sass columns
    line, src = r[0], r[1]
    if not line.isdigit():  # SASS rows under a source line (cuda,sass CSV)
        continue
    try:
        ie = int(r[hdr.index("Instructions Executed")] or 0)
        ss = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    key = (fname, line)
    agg[key][0] += ie
    agg[key][1] += ss
    if not agg[key][2]:
        agg[key][2] = src.strip()[:70]
tot_i = sum(v[0] for v in agg.values())
tot_s = sum(v[1] for v in agg.values())
print(f"total warp-instr {tot_i}  samples {tot_s}")
for (f, l), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f}:{l:>5} {100*i/max(tot_i,1):5.1f}%i {100*s/max(tot_s,1):5.1f}%s  {src}")
