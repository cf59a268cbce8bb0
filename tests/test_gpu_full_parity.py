"""Whole-batch parity at the headline size (opt-in: DSFFT_FULL_PARITY=1).

BASELINE configs[1]: every one of the 2^20 fp16 transforms (and 2^19 fp32)
of N=1024 dual-select, run by the product as ONE batched launch on the
device, compared bit for bit with the reference's own forward
(oracle/_ref, all host cores) in chunks.  Inputs are the bench's synthetic
batch (dsfft_fill_uniform, global-index keyed).  Takes a few minutes of host
CPU; writes a summary to $DSFFT_FULL_PARITY_OUT (default
gpurun_out/full_parity_<precision>.json)."""
import json
import os
import time

import numpy as np
import pytest

from helpers import bit_mismatches

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(os.environ.get("DSFFT_FULL_PARITY") != "1",
                                 reason="opt-in: DSFFT_FULL_PARITY=1")]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("precision,batch", [("fp16", 1 << 20), ("fp32", 1 << 19)])
def test_whole_headline_batch_bit_exact(dsfft, cuda, orc, precision, batch):
    import oracle
    torch = cuda
    chk = oracle.load_ref() if oracle.ref_available() else orc
    n = 1024
    plan = dsfft.make_plan(n, "dual", precision)
    x = dsfft.synthetic_batch(n, 0, batch, 20260419, precision)
    y = dsfft.forward(plan, x)  # one launch over the whole batch
    torch.cuda.synchronize()
    chunk = 1 << 15
    bad = 0
    t0 = time.time()
    for b0 in range(0, batch, chunk):
        xs = x[b0:b0 + chunk].cpu().numpy()
        ys = y[b0:b0 + chunk].cpu().numpy()
        want = chk.forward(xs.astype(np.float64).view(np.complex128)[..., 0], "dual", precision)
        want_w = want.view(np.float64).reshape(ys.shape).astype(ys.dtype)
        bad += bit_mismatches(ys, want_w)
    secs = time.time() - t0
    out = os.environ.get("DSFFT_FULL_PARITY_OUT",
                         os.path.join(ROOT, "gpurun_out", f"full_parity_{precision}.json"))
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump({"n": n, "precision": precision, "strategy": "dual", "transforms": batch,
                   "components_compared": int(batch * n * 2), "mismatches": int(bad),
                   "checker": chk.prefix, "host_cores": os.cpu_count(),
                   "checker_seconds": secs, "launches": 1,
                   "inputs": "dsfft_fill_uniform seed 20260419 (bench.py's batch)"}, f, indent=1)
    assert bad == 0, f"{bad} mismatching components"
