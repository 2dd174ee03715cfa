#!/usr/bin/env python
"""Summarise an ncu --set full capture and a gpu__time_duration launch list into profiles/.

    python tools/summarize_ncu.py <prof.ncu-rep> <launches.csv> <tag>

Writes profiles/<tag>_ncu_summary.txt, profiles/<tag>_launches.txt and updates
profiles/ncu_traffic.json (per-launch DRAM traffic of the attention kernels, read by bench.py).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
]
NAMES = {"jfa_fwd": "jagged_flash_attention_forward", "jfa_bwd": "jagged_flash_attention_backward"}


def to_bytes(v, unit):
    m = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v) * m.get(unit, 1)


def main():
    rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    os.makedirs(PROF, exist_ok=True)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = [f"# ncu --set full summary ({os.path.basename(rep)}), one launch per kernel", ""]
    traffic = {}
    tp = os.path.join(PROF, "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp))
    for d in data:
        name = d[hdr.index("Kernel Name")]
        out.append(f"## {name[:100]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"  {k:70s} {d[i]:>16s} {units[i]}")
        rb = to_bytes(d[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
        wb = to_bytes(d[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
        out.append(f"  {'dram traffic per launch (read + write)':70s} {rb + wb:16.4e} byte")
        out.append("")
        for short, api in NAMES.items():
            if short in name:
                traffic[api] = {"bytes_per_launch": rb + wb, "dram_read": rb, "dram_write": wb,
                                "source": f"profiles/{tag}_ncu_summary.txt"}
    open(os.path.join(PROF, f"{tag}_ncu_summary.txt"), "w").write("\n".join(out) + "\n")
    json.dump(traffic, open(tp, "w"), indent=1)

    agg = defaultdict(list)
    for r in csv.DictReader(l for l in open(launches) if not l.startswith("==")):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            agg[r["Kernel Name"].split("(")[0][:70]].append(float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1))
    lines = [f"# ncu launch list ({os.path.basename(launches)}): gpu__time_duration per kernel, --clock-control none",
             "# (cold-cache, serialised; compare shares, not absolutes)", "",
             f"{'kernel':72s} {'launches':>8s} {'mean us':>10s} {'total us':>10s}"]
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k:72s} {len(v):8d} {sum(v) / len(v):10.1f} {sum(v):10.1f}   {100 * sum(v) / tot:5.1f}%")
    open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    print("\n".join(out))


if __name__ == "__main__":
    main()
