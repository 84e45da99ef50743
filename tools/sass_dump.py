"""Print the hot SASS of an ncu source-page CSV in address order:
    python tools/sass_dump.py file.csv [min_exec] [start] [count]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
iE = hdr.index("Instructions Executed")
iS = hdr.index("Warp Stall Sampling (All Samples)")
mn = int(sys.argv[2]) if len(sys.argv) > 2 else 1
start = int(sys.argv[3]) if len(sys.argv) > 3 else 0
count = int(sys.argv[4]) if len(sys.argv) > 4 else 10 ** 9
n = 0
for r in data:
    e = int(r[iE] or 0)
    if e >= mn:
        if start <= n < start + count:
            print(n, r[0][-5:], e, r[iS], " ".join(r[1].split())[:100])
        n += 1
print("instructions:", n)
