#!/bin/bash
# Launch-shape sweep of the single kernel: fp16 layout x ring depth, fp32 ring
# depth, at >= 4 GiB per step -> gpurun_out/autotune.jsonl (one line per run:
# {"n", "precision", "env", "frac"}).  Defaults in csrc/inst_small.cu come from it.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
out=gpurun_out/autotune.jsonl
: > "$out"
for rep in $(seq ${REPS:-1}); do
for n in ${NS:-64 128 256 512 1024 2048 4096 8192}; do
  for p in fp16 fp32; do
    sb=$([ "$p" = fp16 ] && echo 4 || echo 8)
    b=$(( (4 << 30) / (n * sb) ))
    if [ "$p" = fp16 ]; then envs="1:1 1:2 1:3 1:4 2:1 2:2 2:3 2:4"; else envs="0:1 0:2 0:3 0:4"; fi
    for e in $envs; do
      lay=${e%%:*}; st=${e##*:}
      f=$( ( [ "$lay" = 0 ] && env DSFFT_STAGES=$st python bench.py --n $n --precision $p --batch $b \
               --steps ${STEPS:-20} --warmup 3 --no-cpu --no-e2e --no-accuracy \
             || env DSFFT_F16_LAYOUT=$lay DSFFT_STAGES=$st python bench.py --n $n --precision $p \
               --batch $b --steps ${STEPS:-20} --warmup 3 --no-cpu --no-e2e --no-accuracy ) 2>/dev/null \
           | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['roofline']['frac'])" 2>/dev/null)
      echo "{\"n\": $n, \"precision\": \"$p\", \"layout\": $lay, \"stages\": $st, \"frac\": ${f:-null}}" >> "$out"
    done
  done
done
done
wc -l "$out"
