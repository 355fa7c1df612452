#!/usr/bin/env python
"""Warp-stall reasons per CUDA source line, restricted to a line range (for
one warp role of a warp-specialized kernel).  Usage:
  python tools/ncu_stalls.py report.ncu-rep file.cuh first_line last_line [top]"""
import csv
import io
import os
import subprocess
import sys


def main():
    rep, fsel, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 20
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, hdr, rows, tot = "?", None, [], {}
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = os.path.basename(rec[1])
            continue
        if rec[0] == "Line No":
            hdr = rec
            continue
        if hdr is None or rec[0] in ("", "Function Name") or fname != fsel:
            continue
        ln = int(rec[0])
        if not lo <= ln <= hi:
            continue
        d = dict(zip(hdr[2:], rec[2:]))
        st = {k[6:]: float(v or 0) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k}
        for k, v in st.items():
            tot[k] = tot.get(k, 0) + v
        rows.append((sum(st.values()), ln, rec[1].strip()[:70], st))
    s = sum(tot.values()) or 1
    print("role total:", ", ".join(f"{k} {100 * v / s:.0f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
    for n, ln, src, st in sorted(rows, key=lambda r: -r[0])[:top]:
        top3 = ", ".join(f"{k} {v:.0f}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3])
        print(f"{100 * n / s:5.1f}% L{ln}: {src}  [{top3}]")


if __name__ == "__main__":
    main()
