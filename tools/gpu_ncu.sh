#!/bin/bash
# One `ncu --set full` capture per workload (run under gpurun; one GPU).
#   tools/gpu_ncu.sh "label:--n 4096" "label2:--n 2048 --precision fp32" ...
# Each workload first runs plain (must exit 0), then once under ncu, capturing
# the 4th launch of the kernel family given by KREGEX (default fft_small).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for spec in "$@"; do
  label=${spec%%:*}
  args=${spec#*:}
  cmd="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-accuracy --sustained-seconds 0 $args"
  if timeout 300 $cmd > "gpurun_out/plain_$label.log" 2>&1; then
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-fft_small}" \
      -s "${SKIP:-3}" -c "${COUNT:-1}" -o "gpurun_out/prof_$label" -f $cmd > "gpurun_out/ncu_$label.log" 2>&1
    echo "$label ncu rc=$? $(tail -1 gpurun_out/plain_$label.log | cut -c1-200)"
  else
    echo "$label plain run failed"; tail -5 "gpurun_out/plain_$label.log"
  fi
done
