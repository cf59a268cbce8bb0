#!/usr/bin/env python
"""Format gpurun_out/sweep.jsonl (tools/gpu_sweep.sh) as markdown tables:
% of the measured HBM roofline and transforms/s per (N, precision, strategy).

  python tools/sweep_table.py gpurun_out/sweep.jsonl > profiles/rNN_sweep.md
"""
import json
import sys


def main(path):
    rows = [json.loads(line) for line in open(path) if line.strip().startswith("{")]
    table = {}
    for d in rows:
        c = d["config"]
        table[(c["n"], c["precision"], c["strategy"])] = d
    ns = sorted({k[0] for k in table})
    strats = [s for s in ("standard", "lf", "cosine", "dual") if any(k[2] == s for k in table)]
    clocks = sorted({d.get("clocks", {}).get("sm_mhz") for d in rows} - {None})
    print("| N | precision | " + " | ".join(strats) + " | reference CPU, dual (16 cores) | GPU / CPU |")
    print("|---|---|" + "---|" * len(strats) + "---|---|")
    for n in ns:
        for p in ("fp16", "fp32"):
            cells = []
            for s in strats:
                d = table.get((n, p, s))
                if d is None:
                    cells.append("")
                    continue
                cells.append(f"{100 * d['roofline']['frac']:.1f}% ({d['value'] / 1e6:.1f} M/s)")
            ref = table.get((n, p, "dual"), {}).get("cpu_baseline") or {}
            if ref.get("value"):
                g = table[(n, p, "dual")]["value"]
                cells += [f"{ref['value']:.3g} /s ({ref.get('kind')})", f"{g / ref['value']:.3g}x"]
            else:
                cells += ["", ""]
            if any(cells):
                print(f"| {n} | {p} | " + " | ".join(cells) + " |")
    print()
    print(f"Cells: achieved HBM bandwidth (2 x N x sizeof(complex) per transform) as % of "
          f"the measured copy peak, and transforms/s.  SM clocks under load (MHz): {clocks}.")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep.jsonl")
