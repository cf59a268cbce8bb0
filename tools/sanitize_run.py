#!/usr/bin/env python
"""Small driver touching every kernel family once (single kernel for each
size class and value layout, multipass 2- and 3-group, fp64 passes, error
harness, host pipeline), for `compute-sanitizer --tool <memcheck|racecheck|
synccheck>` runs (one tool per gpurun call).  Exits non-zero on a parity miss.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2604_00567_b200 as dsfft  # noqa: E402
from helpers import bit_mismatches, ref_inputs, to_work  # noqa: E402


def main():
    orc = oracle.load_oracle()
    chk = oracle.load_ref() if oracle.ref_available() else orc
    cases = [(2, "fp16", 3), (8, "fp32", 5), (64, "fp16", 9), (256, "fp16", 5),
             (1024, "fp16", 5), (1024, "fp32", 3), (2048, "fp16", 3), (4096, "fp16", 3),
             (4096, "fp32", 2), (8192, "fp16", 2), (1 << 16, "fp32", 2), (1 << 19, "fp16", 1),
             (256, "fp64", 3)]
    bad = 0
    for n, p, batch in cases:
        for inverse in (False, True):
            x = ref_inputs(orc, n, batch, seed=n, precision=p)
            xw = x if p == "fp64" else to_work(x, p)
            plan = dsfft.make_plan(n, "dual", p)
            y = dsfft.execute(plan, int(inverse), torch.from_numpy(np.ascontiguousarray(xw)).cuda())
            torch.cuda.synchronize()
            want = (chk.inverse if inverse else chk.forward)(x, "dual", p)
            got = y.cpu().numpy()
            if p == "fp64":
                miss = bit_mismatches(got.view(np.float64), want.view(np.float64))
            else:
                miss = bit_mismatches(got, to_work(want, p))
            print(n, p, batch, "inv" if inverse else "fwd", "mismatches", miss, flush=True)
            bad += miss
    rep = dsfft.error_device(dsfft.make_plan(1024, "dual", "fp16"),
                             torch.from_numpy(to_work(ref_inputs(orc, 1024, 4, 1, "fp16"),
                                                      "fp16")).cuda(), "forward")
    print("error harness", rep, flush=True)
    xh = to_work(ref_inputs(orc, 512, 7, 2, "fp32"), "fp32")
    yh = np.empty_like(xh)
    dsfft.execute_host(dsfft.make_plan(512, "lf", "fp32"), 0, xh, yh, 7)
    bad += bit_mismatches(yh, to_work(chk.forward(ref_inputs(orc, 512, 7, 2, "fp32"), "lf",
                                                  "fp32"), "fp32"))
    print("total mismatches", bad)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
