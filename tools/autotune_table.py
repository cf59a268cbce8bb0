#!/usr/bin/env python
"""Summarise gpurun_out/autotune.jsonl (tools/gpu_autotune.sh): mean % of HBM
per (N, precision, fp16 layout, ring depth) over the repeats, best marked.

  python tools/autotune_table.py gpurun_out/autotune.jsonl
"""
import collections
import json
import sys


def main(path):
    acc = collections.defaultdict(list)
    for line in open(path):
        d = json.loads(line)
        if d["frac"] is not None:
            acc[(d["n"], d["precision"], d["layout"], d["stages"])].append(d["frac"])
    keys = sorted({(n, p) for n, p, _, _ in acc})
    print("| N | precision | " + " | ".join(["P S1", "P S2", "P S3", "P S4", "C S1", "C S2",
                                            "C S3", "C S4"]) + " |")
    print("|---|---|" + "---|" * 8)
    for n, p in keys:
        cells = {}
        for (n2, p2, lay, st), v in acc.items():
            if (n2, p2) == (n, p):
                cells[(lay, st)] = sum(v) / len(v)
        best = max(cells, key=cells.get)
        row = []
        for lay in ((1, 2) if p == "fp16" else (0,)):
            for st in (1, 2, 3, 4):
                v = cells.get((lay, st))
                txt = "" if v is None else f"{100 * v:.1f}"
                row.append(f"**{txt}**" if (lay, st) == best else txt)
        if p == "fp32":
            row += [""] * 4
        print(f"| {n} | {p} | " + " | ".join(row) + " |")
    print("\nfp32 rows list ring depths 1-4 in the first four columns.")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/autotune.jsonl")
