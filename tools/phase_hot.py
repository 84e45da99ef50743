"""Group an ncu `--print-source cuda,sass` CSV by phases given as
name=first-last line ranges of one file: python tools/phase_hot.py CSV FILE name=a-b ..."""
import csv
import sys
from collections import defaultdict

path, fname_sel = sys.argv[1], sys.argv[2]
ranges = []
for a in sys.argv[3:]:
    name, rng = a.split("=")
    lo, hi = map(int, rng.split("-"))
    ranges.append((name, lo, hi))
rows = list(csv.reader(open(path)))
fname, hdr = "", None
agg = defaultdict(lambda: [0, 0])
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0]:
        continue
    try:
        ie = int(r[hdr.index("Instructions Executed")] or 0)
        ss = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    line = int(r[0])
    key = fname
    if fname == fname_sel:
        key = next((n for n, lo, hi in ranges if lo <= line <= hi), f"{fname}:other")
    agg[key][0] += ie
    agg[key][1] += ss
ti = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:28s} inst {100 * v[0] / ti:5.1f}%  stall {100 * v[1] / ts:5.1f}%")
