#!/bin/bash
# Multipass launch-shape sweep: tile groups x ring depth (x fp16 layout) at
# 1 GiB per step -> gpurun_out/autotune_mp.jsonl.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
out=gpurun_out/autotune_mp.jsonl
: > "$out"
for rep in $(seq ${REPS:-1}); do
for n in ${NS:-16384 65536 262144 1048576}; do
  for p in fp16 fp32; do
    lays=$([ "$p" = fp16 ] && echo "1 2" || echo "1")
    for lay in $lays; do for g in 1 2; do for st in 1 2; do
      f=$(env DSFFT_MP_F16_LAYOUT=$lay DSFFT_MP_GROUPS=$g DSFFT_MP_STAGES=$st python bench.py --n $n \
            --precision $p --steps ${STEPS:-20} --warmup 3 --no-cpu --no-e2e --no-accuracy 2>/dev/null \
          | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['roofline']['frac'])" 2>/dev/null)
      echo "{\"n\": $n, \"precision\": \"$p\", \"layout\": $lay, \"groups\": $g, \"stages\": $st, \"frac\": ${f:-null}}" >> "$out"
    done; done; done
  done
done
done
wc -l "$out"
