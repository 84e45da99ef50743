"""Summarise an ncu source-page SASS CSV (tools/ncu_source.sh): warp
instructions per key by opcode, stall reasons, hottest instructions.
    python tools/sass_profile.py file.csv [nkeys_log2]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
nk = 2 ** int(sys.argv[2]) if len(sys.argv) > 2 else 2 ** 28
hdr, data = rows[1], rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
print(rows[0][1][:120])
tot = sum(int(r[iE] or 0) for r in data)
print(f"warp-inst/key {tot / nk:.3f}")
ops, opsS = collections.Counter(), collections.Counter()
for r in data:
    t = r[1].strip().split()
    if not t:
        continue
    o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    ops[o] += int(r[iE] or 0)
    opsS[o] += int(r[iS] or 0)
print(" ".join(f"{o}:{c / nk:.3f}" for o, c in ops.most_common(16)))
stall = collections.Counter()
for r in data:
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                stall[h] += int(r[i])
            except ValueError:
                pass
ts = sum(stall.values()) or 1
print("stalls:", " ".join(f"{k[6:]}:{v / ts:.2f}" for k, v in stall.most_common(8)))
byc = collections.Counter()
for r in data:
    e = int(r[iE] or 0)
    byc[e] += e
print("exec-count groups (count, warp-inst/key):", [(c, round(s / nk, 3)) for c, s in byc.most_common(6)])
