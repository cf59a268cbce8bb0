#!/bin/bash
# all GPU tests + headline bench + a large-N sweep (numbers only)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
b() { # label args...
  local label=$1; shift
  timeout 300 python bench.py --steps ${STEPS:-20} --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/b_$label.log 2>&1
  echo "$label: $(python -c "import json; d=json.loads(open('gpurun_out/b_$label.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['value']/1e6,1), 'M/s frac', round(d['roofline']['frac'],4), 'launches', d['gpu_launches'])" 2>&1 | tail -1)"
}
b n1024_fp16
b n1024_fp32 --precision fp32
for n in ${NS:-256 4096 65536 1048576}; do b n${n}_fp16 --n $n; b n${n}_fp32 --n $n --precision fp32; done
