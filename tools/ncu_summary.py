#!/usr/bin/env python
"""Summarise an ncu report (run here, no GPU needed): key throughput /
traffic / pipe metrics and the top warp-stall reasons per kernel, as
markdown.  Usage: python tools/ncu_summary.py report.ncu-rep [title]"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tc pipe active %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem LSU wavefronts"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum", "smem tensor-core wavefronts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (occupancy)"),
    ("smsp__inst_executed.sum", "instructions"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    out = [f"# {title}", "", f"Source report: `{rep}` (ncu --set full --clock-control none).", ""]
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        out.append(f"## `{name[:110]}`")
        out.append("")
        out.append("| metric | value |")
        out.append("|---|---|")
        for k, label in KEYS:
            if k in col and r[col[k]] != "":
                out.append(f"| {label} (`{k}`) | {r[col[k]]} {units[col[k]]} |")
        st = [(h, float(r[i])) for h, i in col.items()
              if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued") and r[i] not in ("",)]
        tot = sum(v for _, v in st) or 1.0
        st.sort(key=lambda t: -t[1])
        out.append("")
        out.append("Top warp-stall samples: " + ", ".join(
            f"{re.sub('smsp__pcsamp_warps_issue_stalled_', '', h)} {100 * v / tot:.0f}%" for h, v in st[:6]))
        out.append("")
    print("\n".join(out))


if __name__ == "__main__":
    main()
