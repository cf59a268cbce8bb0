#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
b() { local label=$1; shift
  env $ENVS timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/b_$label.log 2>&1
  echo "$label $ENVS: $(python -c "import json; d=json.loads(open('gpurun_out/b_$label.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), d['gpu_launches'])" 2>&1 | tail -1)"; }
for c in 24 48 96 256 1100; do
  ENVS="DSFFT_MP_CHUNK_MB=$c" b n65536_c$c --n 65536
  ENVS="DSFFT_MP_CHUNK_MB=$c" b n1m_c$c --n 1048576
  ENVS="DSFFT_MP_CHUNK_MB=$c" b n65536_f32_c$c --n 65536 --precision fp32
done
