#!/usr/bin/env python
"""Aggregate ncu warp-stall samples by CUDA source line (needs -lineinfo + --import-source on).

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep jfa_fwd [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", f"regex:{kern}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, lines = "?", None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit() or len(r) != len(hdr):
            continue
        if r[2] != "-":  # per-SASS rows; keep per-line aggregates only
            continue
        rec = dict(zip(range(len(hdr)), r))
        samples = int(r[4] or 0)
        if samples == 0:
            continue
        reasons = {hdr[i]: int(r[i]) for i in range(len(hdr)) if hdr[i].startswith("stall_") and
                   "Not Issued" not in hdr[i] and r[i].isdigit() and int(r[i]) > 0}
        lines.append((samples, fname, int(r[0]), r[1].strip()[:80], reasons))
        del rec
    tot = sum(x[0] for x in lines)
    print(f"total samples {tot}")
    for s, f, ln, src, rs in sorted(lines, reverse=True)[:top]:
        rr = ", ".join(f"{k[6:]}={v}" for k, v in sorted(rs.items(), key=lambda kv: -kv[1])[:3])
        print(f"{s:7d} {100 * s / tot:5.1f}% {f}:{ln:<5d} {src:80s} | {rr}")


if __name__ == "__main__":
    main()
