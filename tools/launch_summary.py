"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel:
launches, summed device time and share.   python tools/launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "").replace("ams::<unnamed>::", "")
    v = float(r[vi].replace(",", ""))
    v = v / 1e3 if r[ui] == "ns" else v * (1e3 if r[ui] == "ms" else 1)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print("| kernel | launches | device time (us, ncu serial) | share |\n|---|---|---|---|")
for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{name[:110]}` | {n} | {us:.1f} | {100 * us / tot:.1f}% |")
