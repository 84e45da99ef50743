"""Static SASS opcode counts of the hot kernels in the built library
(cuobjdump -sass): which load / store / staging / vote / atomic instructions
each kernel is made of.

    python tools/sass_ops.py > profiles/<round>_sass_ops.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_1410_6754_b200", "lib", "obj")
HOT = [("k_hist.cu.o", "k_histILi0ELb0ELb1ELi1ELb0ELi1E", "k_hist level 1 (u64, min/max, ids, plain)"),
       ("k_hist.cu.o", "k_histILi0ELb0ELb0ELi1ELb0ELi1E", "k_hist level 2 (u64, ids, plain)"),
       ("k_scatter.cu.o", "k_scatterILi0ELi2ELb0ELi0ELb0E", "k_scatter stable (ids, keys only)"),
       ("k_scatter.cu.o", "k_scatterILi0ELi2ELb0ELi2ELb0E", "k_scatter unstable (ids, keys only)"),
       ("k_scatter.cu.o", "k_scatterILi0ELi2ELb0ELi0ELb1E", "k_scatter stable, peer destinations"),
       ("k_final.cu.o", "k_scatter_fixedILi0E", "k_scatter_fixed"),
       ("k_final.cu.o", "k_cell_sort_fixedILi0E", "k_cell_sort_fixed (u64 out)"),
       ("k_final.cu.o", "k_smem_sortILi0ELb1E", "k_smem_sort (u64, payloads)")]
WATCH = ["LDG", "LDG.E.128", "LDGSTS", "UBLKCP", "SYNCS", "STG", "STG.E.128", "LDS", "LDS.128", "STS", "STS.128",
         "ATOMS", "ATOMG", "RED", "VOTE", "SHFL", "BAR", "MATCH", "IMAD", "LOP3"]


def kernels(obj):
    txt = subprocess.run(["cuobjdump", "-sass", os.path.join(OBJ, obj)], capture_output=True, text=True).stdout
    out, name = collections.defaultdict(list), None
    for ln in txt.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            name = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(.*?);", ln)
        if m and name:
            t = m.group(1).split()
            out[name].append(t[1] if t[0].startswith("@") else t[0])
    return out


print("# Static SASS opcode counts of the hot kernels (cuobjdump -sass of the built objects, sm_100a)\n")
print("`UBLKCP` = bulk (TMA-engine) global->shared copy, `LDGSTS` = cp.async, `SYNCS` = mbarrier ops,")
print("`*.128` = 16-byte accesses.  Counts are static instructions, not executed ones.\n")
print("| kernel | total | " + " | ".join(WATCH) + " |")
print("|---|---|" + "---|" * len(WATCH))
cache = {}
for obj, pat, label in HOT:
    ks = cache.setdefault(obj, kernels(obj))
    hit = [k for k in ks if pat in k]
    if not hit:
        print(f"| {label} | not found |")
        continue
    ops = ks[hit[0]]
    cnt = collections.Counter()
    for o in ops:
        base = o.split(".")[0]
        cnt[base] += 1
        if ".128" in o:
            cnt[base + (".E.128" if base in ("LDG", "STG") else ".128")] += 1
    print(f"| {label} | {len(ops)} | " + " | ".join(str(cnt.get(w, 0)) for w in WATCH) + " |")
