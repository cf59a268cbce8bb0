#!/usr/bin/env python
"""Summarise ncu captures (gpurun_out/*.ncu-rep, launch-list CSVs) into
profiles/: a JSON keyed by workload (read by bench.py for roofline.traffic)
and a markdown table per capture.

  python tools/ncu_summary.py --rep gpurun_out/prof_n1024_fp16.ncu-rep \
      --key n1024_fp16_dual --batch 1048576 --round r01 [--launches gpurun_out/launches_fp16.csv]
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.sum", "sm__inst_executed_pipe_alu.sum",
    "sm__inst_executed_pipe_lsu.sum", "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg",
    "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_selected",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_mio_throttle",
    "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_not_selected",
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = vals[i].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                d[m] = (v, units[i])
        res.append(d)
    return res


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return v * scale.get(unit, 1)


def to_ms(v, unit):
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1, "s": 1e3}
    return v * scale.get(unit, 1)


def launch_shares(path):
    """Per-kernel share of device time from a --metrics gpu__time_duration.sum list."""
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    tot, per = 0.0, {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        t = to_ms(float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
        name = r["Kernel Name"].split("<")[0].split("(")[0][:60]
        per[name] = per.get(name, 0.0) + t
        tot += t
    return {k: {"ms": v, "share": v / tot if tot else 0.0} for k, v in per.items()}, len(rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--key", required=True)
    ap.add_argument("--batch", type=int, required=True)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--sample-bytes", type=int, default=4)
    ap.add_argument("--round", default="r01")
    ap.add_argument("--launches", default=None)
    ap.add_argument("--kernel", default="fft", help="substring of the captured kernel's name")
    a = ap.parse_args()
    ms = raw_metrics(a.rep)
    k = [m for m in ms if a.kernel in m["kernel"]][0]
    rd = to_bytes(*k["dram__bytes_read.sum"])
    wr = to_bytes(*k["dram__bytes_write.sum"])
    dur = to_ms(*k["gpu__time_duration.sum"])
    algo = 2.0 * a.n * a.sample_bytes * a.batch
    summary = {
        "kernel": k["kernel"][:160], "batch": a.batch, "n": a.n, "duration_ms_under_ncu": dur,
        "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes": rd + wr,
        "algorithmic_bytes": algo, "traffic_over_algorithmic": (rd + wr) / algo,
        "metrics": {m: k[m][0] for m in METRICS if m in k},
        "source": os.path.relpath(a.rep, ROOT),
    }
    if a.launches:
        shares, nrows = launch_shares(a.launches)
        summary["launch_list"] = shares
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    jpath = os.path.join(ROOT, "profiles", "ncu_summary.json")
    allj = json.load(open(jpath)) if os.path.exists(jpath) else {}
    allj[a.key] = summary
    json.dump(allj, open(jpath, "w"), indent=1, sort_keys=True)
    md = os.path.join(ROOT, "profiles", f"{a.round}_{a.key}.md")
    with open(md, "w") as f:
        f.write(f"# ncu --set full: {a.key} ({a.round})\n\n")
        f.write(f"kernel `{summary['kernel']}`\n\n| metric | value |\n|---|---|\n")
        f.write(f"| duration (under ncu, cold) | {dur:.4f} ms |\n")
        f.write(f"| dram read / write | {rd/1e9:.4f} / {wr/1e9:.4f} GB |\n")
        f.write(f"| algorithmic bytes | {algo/1e9:.4f} GB (traffic/algorithmic "
                f"{(rd+wr)/algo:.4f}) |\n")
        for m in METRICS:
            if m in k:
                f.write(f"| {m} | {k[m][0]} {k[m][1]} |\n")
        if a.launches:
            f.write("\n## launch list (share of device time)\n\n| kernel | ms | share |\n|---|---|---|\n")
            for name, v in sorted(summary["launch_list"].items(), key=lambda kv: -kv[1]["ms"]):
                f.write(f"| {name} | {v['ms']:.4f} | {v['share']:.3f} |\n")
    print(json.dumps({a.key: {x: summary[x] for x in ("dram_bytes", "algorithmic_bytes",
                                                      "traffic_over_algorithmic")}}))


if __name__ == "__main__":
    main()
