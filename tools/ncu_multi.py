#!/usr/bin/env python
"""Markdown summary of every kernel in an ncu report (multi-launch captures,
e.g. the pass-group launches of one multipass step).

  python tools/ncu_multi.py gpurun_out/prof_X.ncu-rep "title" > profiles/rNN_X.md
"""
import csv
import subprocess
import sys

ROWS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma_type_fp16.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "launch__shared_mem_per_block_dynamic",
]


def main(rep, title):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    print(f"# {title}\n")
    print(f"Source: `{rep}` (`ncu --set full --clock-control none`).\n")
    for v in rows[2:]:
        print(f"## `{v[h.index('Kernel Name')][:110]}`\n")
        print("| metric | value |\n|---|---|")
        for m in ROWS:
            if m in h:
                i = h.index(m)
                print(f"| {m} | {v[i]} {units[i]} |")
        st = sorted(((float(v[i]), c.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                     for i, c in enumerate(h)
                     if c.startswith("smsp__pcsamp_warps_issue_stalled_")
                     and not c.endswith("not_issued") and v[i].replace(".", "", 1).isdigit()),
                    reverse=True)
        print("| top stall samples | " + ", ".join(f"{n} {int(x)}" for x, n in st[:8]) + " |\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
