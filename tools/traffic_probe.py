"""DRAM traffic per launch across the large-N paths (run under ncu):

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
      --csv --log-file gpurun_out/traffic.csv python tools/traffic_probe.py

Each config runs one forward over 256 MiB of input; the printed order maps
the launches in the ncu log to configs (algorithmic bytes = 256 MiB read +
256 MiB written per pass group for the two-launch path)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_00567_b200 as dsfft  # noqa: E402

CONFIGS = [(m, p) for m in (14, 16, 17, 18, 19, 20, 22, 24) for p in ("fp16", "fp32")]

for m, prec in CONFIGS:
    n = 1 << m
    sb = 4 if prec == "fp16" else 8
    batch = max(2, (256 << 20) // (n * sb))
    plan = dsfft.make_plan(n, "dual", prec)
    x = dsfft.synthetic_batch(n, 0, batch, 1, prec)
    y = dsfft.forward(plan, x)
    torch.cuda.synchronize()
    print(f"config m={m} {prec} batch={batch} launches={dsfft.last_launch_count()}", flush=True)
    del x, y
