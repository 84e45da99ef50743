"""Per-source-line totals of an ncu SASS source page (tools/ncu_source.sh)
when the CUDA-correlated page carries no metrics: the line of every SASS
instruction comes from `nvdisasm -g` of the object file, aligned with the
ncu rows by opcode sequence.

    python tools/sass_lines.py k1_sass.csv paper_1410_6754_b200/lib/obj/k_scatter.cu.o 'k_scatterILi0ELi2ELb0ELi0ELb0E' [top] [log2n]
"""
import collections
import csv
import difflib
import os
import re
import subprocess
import sys
import tempfile

csv_path, obj, pat = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
nk = 2 ** (int(sys.argv[5]) if len(sys.argv) > 5 else 28)

with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, check=True,
                   stdout=subprocess.DEVNULL)
    cubin = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(td, cubin)], capture_output=True,
                         text=True).stdout.splitlines()
ins, cur, on = [], None, False
for ln in dis:
    if ln.startswith(".text."):
        on = pat in ln
        continue
    if not on:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(.*?);", ln)
    if m:
        t = m.group(1).split()
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ins.append((op, cur))
rows = list(csv.reader(open(csv_path)))
hdr, data = rows[1], rows[2:]
iE, iS = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ops = []
for r in data:
    t = r[1].strip().split()
    ops.append((t[1] if t[0].startswith("@") else t[0]).split(".")[0] if t else "")
sm = difflib.SequenceMatcher(None, [o for o, _ in ins], ops, autojunk=False)
line_of = {}
for a, b, n in sm.get_matching_blocks():
    for i in range(n):
        line_of[b + i] = ins[a + i][1]
agg = collections.defaultdict(lambda: [0, 0])
last = None
for j, r in enumerate(data):
    last = line_of.get(j, last)
    agg[last][0] += int(r[iE] or 0)
    agg[last][1] += int(r[iS] or 0)
ti = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values()) or 1
print(f"{len(ins)} disassembled / {len(ops)} profiled instructions, {len(line_of)} aligned; "
      f"warp-inst/key {ti / nk:.3f}")
src_cache = {}
for key, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    text = ""
    if key:
        for root in ("paper_1410_6754_b200/csrc", "."):
            p = os.path.join(root, key[0])
            if os.path.exists(p):
                src_cache.setdefault(p, open(p).read().splitlines())
                text = src_cache[p][key[1] - 1].strip()[:80]
                break
    print(f"{key[0] if key else '?':>16}:{key[1] if key else 0:<5} {i / nk:6.3f} w-i/key {100 * i / ti:5.1f}%i "
          f"{100 * s / ts:5.1f}%s  {text}")
