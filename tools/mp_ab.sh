#!/bin/bash
# A/B of the large-N paths on one GPU: fused one-launch (DSFFT_MP_FUSED=1;
# the default for fp16 2^14/2^16 and fp32 2^14) vs two launches (=0).
# Prints one line per (N, precision, path): ms per step and roofline fraction.
# usage: tools/mp_ab.sh [sizes...]   (run under gpurun)
sizes=${@:-16384 65536 262144}
for n in $sizes; do
  for p in fp16 fp32; do
    for f in 1 0; do
      out=$(DSFFT_MP_FUSED=$f timeout 300 python bench.py --n $n --precision $p --steps 20 \
            --warmup 3 --no-e2e --no-cpu --no-accuracy --sustained-seconds 0 2>&1 | grep '^{')
      python - "$n" "$p" "$f" "$out" <<'PY'
import json, sys
n, p, f, line = sys.argv[1:5]
try:
    d = json.loads(line)
    print(f"N={n:>8} {p} fused={f}: {d['ms_per_step']:.3f} ms/step  frac={d['roofline']['frac']:.3f}  "
          f"batch={d['config']['batch_per_gpu']} launches={d['roofline']['launches_per_step']}")
except Exception as e:
    print(f"N={n} {p} fused={f}: FAILED {line[:200]!r}")
PY
    done
  done
done
