#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
b() { local label=$1; shift
  env $ENVS timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e --no-accuracy "$@" > gpurun_out/b_$label.log 2>&1
  echo "$label $ENVS: $(python -c "import json; d=json.loads(open('gpurun_out/b_$label.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))" 2>&1 | tail -1)"; }
for n in 2 8 32 64 128; do ENVS="" b n${n}_f16 --n $n; ENVS="DSFFT_F16_LAYOUT=1" b n${n}_f16p --n $n; ENVS="" b n${n}_f32 --n $n --precision fp32 --batch $((268435456 / n)); done
C1="python bench.py --n 65536 --steps 1 --warmup 3 --no-cpu --no-e2e --no-accuracy"
$C1 > gpurun_out/mp_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:mp_kernel -s 6 -c 2 -o gpurun_out/prof_mp65536c $C1 > gpurun_out/ncu_mp.log 2>&1; echo ncu_rc=$?
