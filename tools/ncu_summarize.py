"""Summarise one `ncu --set full` capture of tools/profile_case.py (the second
cfg2 sort's hist / scatter / smem_sort launches, tools/ncu_round.sh) into
profiles/ncu_traffic.json (bench.py reads `traffic` from it) and a markdown
table on stdout.

    python tools/ncu_summarize.py gpurun_out/TAG/full_raw.csv [n_keys] [--write]
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# Kernel template -> bench category, in launch order of one cfg2 sort.
CATS = [
    ("k_hist<0, 0, 1", "level_hist (level 1, minmax)"),
    ("k_scatter<0, 2, 0, 0,", "level_scatter"),
    ("k_scatter<0, 0, 0, 0,", "level_scatter"),
    ("k_hist<0, 0, 0", "level_hist (level 2)"),
    ("k_scatter<0, 2, 0, 2,", "level_scatter_unstable"),
    ("k_scatter_u<0, 2>", "level_scatter_unstable"),
    ("k_scatter_u<0, 0>", "level_scatter_unstable"),
    ("k_hist<0, 1", "final_hist"),
    ("k_scatter_fixed<0>", "final_scatter"),
    ("k_scatter_u<0, 1>", "final_scatter"),
    ("k_scatter<0, 1, 0, 2,", "final_scatter"),
    ("k_smem_sort<0, 0", "smem_sort"),
    ("k_cell_sort_fixed<0>", "smem_sort"),
    ("k_bucket_sort", "smem_sort"),
]
ALG = {"smem_sort": 16, "level_scatter": 16, "level_scatter_unstable": 16, "final_scatter": 16,
       "level_hist (level 1, minmax)": 8, "level_hist (level 2)": 8, "final_hist": 8}


def f(r, hdr, name):
    try:
        return float(r[hdr.index(name)])
    except (ValueError, IndexError):
        return float("nan")


def main():
    path = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 1 << 28
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    out = {}
    print("| kernel | template | ncu ms | DRAM read+write (GB) | algorithmic (GB) | ratio | warp-inst/key |"
          " IPC | warps active % | regs |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        cat = next((c for pat, c in CATS if pat in name), None)
        if cat is None:
            continue
        dup_variant = "k_hist<" in name and name.split("(")[0].rstrip().endswith(", 2>")
        if dup_variant:  # the duplicate-heavy half of a histogram launch pair
            cat = cat + " [dup variant, exits]"
        rd = f(r, hdr, "dram__bytes_read.sum") * scale.get(units[hdr.index("dram__bytes_read.sum")], 1)
        wr = f(r, hdr, "dram__bytes_write.sum") * scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
        ms = f(r, hdr, "gpu__time_duration.sum")
        if units[hdr.index("gpu__time_duration.sum")] == "us":
            ms /= 1e3
        inst = f(r, hdr, "smsp__inst_executed.sum")
        alg = 0 if dup_variant else ALG[cat] * n
        tmpl = name.split("(")[0].replace("void ", "")
        rec = {"template": tmpl, "dram_bytes_read": rd, "dram_bytes_write": wr, "traffic": rd + wr,
               "algorithmic_bytes": alg, "traffic_over_algorithmic": (rd + wr) / alg if alg else None,
               "ncu_ms": ms,
               "warp_inst_per_key": inst / n,
               "ipc": f(r, hdr, "sm__inst_executed.avg.per_cycle_active"),
               "warps_active_pct": f(r, hdr, "sm__warps_active.avg.pct_of_peak_sustained_active"),
               "regs": f(r, hdr, "launch__registers_per_thread")}
        key = cat
        i = 2
        while key in out:
            key = f"{cat} #{i}"
            i += 1
        out[key] = rec
        print(f"| {key} | `{tmpl}` | {ms:.3f} | {(rd + wr) / 1e9:.3f} | {alg / 1e9:.3f} | "
              f"{((rd + wr) / alg) if alg else 0:.3f} | {inst / n:.2f} | {rec['ipc']:.2f} | {rec['warps_active_pct']:.0f} | "
              f"{rec['regs']:.0f} |")
    if "--write" in sys.argv:
        d = {"source": "ncu --set full --clock-control none, tools/profile_case.py 28 2 (cfg2: 2^28 u64, "
                       "p=64, (8,8)), second sort, one launch each (tools/ncu_round.sh)",
             "workload": "cfg2", "n_keys": n, "kernels": out}
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as fh:
            json.dump(d, fh, indent=1)


if __name__ == "__main__":
    main()
