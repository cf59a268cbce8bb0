#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest(default) rc=$?"; tail -1 gpurun_out/pytest_gpu.log
DSFFT_F16_LAYOUT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k fp16 > gpurun_out/pytest_gpu_pair.log 2>&1; echo "pytest(pairs) rc=$?"; tail -1 gpurun_out/pytest_gpu_pair.log
run() { # label env...
  local label=$1; shift
  env "$@" timeout 120 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e $EXTRA > gpurun_out/sw_$label.log 2>&1
  echo "$label: $(python -c "import json; d=json.loads(open('gpurun_out/sw_$label.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
}
run pair_s2_g12 DSFFT_F16_LAYOUT=1 DSFFT_STAGES=2 DSFFT_GROUPS=12
for cfg in "2 24" "2 20" "2 16" "3 16" "3 12" "4 12" "4 10" "2 12"; do
  set -- $cfg
  run c_s$1_g$2 DSFFT_F16_LAYOUT=2 DSFFT_STAGES=$1 DSFFT_GROUPS=$2
done
for cfg in "2 12" "3 8"; do set -- $cfg; EXTRA="--precision fp32 --batch 524288" run f32_s$1_g$2 DSFFT_STAGES=$1 DSFFT_GROUPS=$2; done
