"""Summarise an ncu source-page CSV (--page source --print-source sass):
instruction counts per key and the hottest SASS lines by stall samples."""
import csv
import sys

path = sys.argv[1]
nkeys = float(sys.argv[2]) if len(sys.argv) > 2 else 2**28
top_n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = list(csv.reader(open(path)))
hdr = next(r for r in rows if "Source" in r and "Address" in r)
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
src = hdr.index("Source")
data = [r for r in rows if len(r) == len(hdr) and r[si].isdigit()]
tot_s = sum(int(r[si]) for r in data)
tot_i = sum(int(r[ie] or 0) for r in data)
print(f"samples {tot_s}  warp-instr {tot_i}  thread-instr/key {tot_i * 32 / nkeys:.1f}")
ops = {}
for r in data:
    op = r[src].split()[0] if r[src].split() else "?"
    if op.startswith("@"):
        op = r[src].split()[1]
    op = op.split(".")[0]
    a = ops.setdefault(op, [0, 0])
    a[0] += int(r[si]); a[1] += int(r[ie] or 0)
print("by opcode (samples, warp-instr):")
for op, (s, i) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"  {op:10s} {100*s/max(tot_s,1):5.1f}%  {i:10d}")
for r in sorted(data, key=lambda r: -int(r[si]))[:top_n]:
    print(r[si].rjust(6), (r[ie] or "0").rjust(10), r[src][:100])
