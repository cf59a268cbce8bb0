#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "bit_exact_vs_reference" > gpurun_out/pytest_small.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_small.log
DSFFT_F16_LAYOUT=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "bit_exact_vs_reference and fp16" > gpurun_out/pytest_small_c.log 2>&1; echo "pytest f16c rc=$?"; tail -1 gpurun_out/pytest_small_c.log
b() { local label=$1; shift
  env $ENVS timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/b_$label.log 2>&1
  echo "$label $ENVS: $(python -c "import json; d=json.loads(open('gpurun_out/b_$label.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))" 2>&1 | tail -1)"; }
for n in 64 128 256 512 2048 4096; do
  for lay in 1 2; do ENVS="DSFFT_F16_LAYOUT=$lay" b n${n}_f16_l$lay --n $n; done
  ENVS="" b n${n}_f32 --n $n --precision fp32 --batch $((1<<30>>(${#n}>3?0:0)))
done
