#!/bin/bash
# Config-3 / config-5 sweep (BASELINE.json): every N x precision x variant
# through bench.py, one JSON line each -> gpurun_out/sweep.jsonl.
#   tools/gpu_sweep.sh            (run under gpurun; format with tools/sweep_table.py)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
out=gpurun_out/sweep.jsonl
: > "$out"
NS=${NS:-"64 128 256 512 1024 2048 4096 8192"}
LARGE=${LARGE:-"16384 32768 65536 131072 262144 524288 1048576 16777216"}
for n in $NS; do
  for p in fp16 fp32; do
    sb=$([ "$p" = fp16 ] && echo 4 || echo 8)
    batch=$(( (4 << 30) / (n * sb) ))  # >= 4 GiB of input
    for s in ${STRATS:-standard lf cosine dual}; do
      # the reference's CPU path beside it (dual only, a 3 s sample on all cores)
      cpu=$([ "$s" = dual ] && echo "--cpu-seconds 3" || echo "--no-cpu")
      timeout 300 python bench.py --n "$n" --precision "$p" --strategy "$s" --steps "${STEPS:-30}" \
        --warmup 3 --batch "$batch" $cpu --no-e2e --no-accuracy --sustained-seconds 0 \
        2>/dev/null | tail -1 >> "$out"
    done
  done
done
for n in $LARGE; do
  for p in fp16 fp32; do
    for s in ${LSTRATS:-standard dual}; do
      cpu=$([ "$s" = dual ] && echo "--cpu-seconds 3" || echo "--no-cpu")
      timeout 300 python bench.py --n "$n" --precision "$p" --strategy "$s" --steps "${STEPS:-30}" \
        --warmup 3 $cpu --no-e2e --no-accuracy --sustained-seconds 0 2>/dev/null | tail -1 >> "$out"
    done
  done
done
wc -l "$out"
