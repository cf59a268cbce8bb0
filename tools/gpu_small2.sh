#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
b() { local label=$1; shift
  env $ENVS timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/b_$label.log 2>&1
  echo "$label $ENVS: $(python -c "import json; d=json.loads(open('gpurun_out/b_$label.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))" 2>&1 | tail -1)"; }
for n in 2048 4096; do
  for lay in 1 2; do for st in 1 2 3; do ENVS="DSFFT_F16_LAYOUT=$lay DSFFT_STAGES=$st" b n${n}_f16_l${lay}_s$st --n $n; done; done
  for st in 1 2 3; do ENVS="DSFFT_STAGES=$st" b n${n}_f32_s$st --n $n --precision fp32 --batch 262144; done
done
for n in 64 128 256 512 1024; do
  for st in 2 3 4; do ENVS="DSFFT_F16_LAYOUT=2 DSFFT_STAGES=$st" b n${n}_f16c_s$st --n $n; done
  for st in 2 3 4; do ENVS="DSFFT_STAGES=$st" b n${n}_f32_s$st --n $n --precision fp32 --batch $((268435456 / n)); done
done
