#!/bin/bash
# parity + launch-shape sweep for the headline config
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
PREC=${PREC:-fp16}
for cfg in ${SWEEP:-"2 8" "2 12" "2 16" "3 8" "3 10" "4 6" "4 8"}; do
  set -- $cfg
  DSFFT_STAGES=$1 DSFFT_GROUPS=$2 timeout 120 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e --precision $PREC $EXTRA > gpurun_out/sw_s$1_g$2.log 2>&1
  echo "S=$1 G=$2: $(python -c "import json; d=json.loads(open('gpurun_out/sw_s$1_g$2.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
done
