#!/usr/bin/env python
"""Per-source-line hot spots of an ncu report (needs -lineinfo builds):
instructions executed and warp-stall samples aggregated by CUDA source line
(ncu --page source --print-source cuda,sass).
Usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import os
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, fname, hdr = [], "?", None
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = os.path.basename(rec[1])
            continue
        if rec[0] == "Line No":
            hdr = rec
            continue
        if hdr is None or rec[0] in ("", "Function Name"):
            continue
        d = dict(zip(hdr[2:], rec[2:]))  # the second "Source" column duplicates
        try:
            ins = float(d.get("Instructions Executed") or 0)
            smp = float(d.get("Warp Stall Sampling (All Samples)") or 0)
        except ValueError:
            continue
        if ins or smp:
            rows.append((ins, smp, f"{fname}:{rec[0]}", rec[1].strip()[:80]))
    tot_i = sum(r[0] for r in rows) or 1
    tot_s = sum(r[1] for r in rows) or 1
    print(f"total warp-instructions {tot_i:.3e}, stall samples {tot_s:.0f}")
    for ins, smp, ln, src in sorted(rows, key=lambda r: -r[1])[:top]:
        print(f"{100 * ins / tot_i:5.1f}% ins {100 * smp / tot_s:5.1f}% smp  {ln}: {src}")


if __name__ == "__main__":
    main()
