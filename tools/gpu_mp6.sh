#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x -m gpu -p no:cacheprovider -k "multipass or many_streams or random or graph" > gpurun_out/pytest_mp.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_mp.log
b() { local label=$1; shift
  env $ENVS timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-accuracy "$@" > gpurun_out/b_$label.log 2>&1
  echo "$label $ENVS: $(python -c "import json; d=json.loads(open('gpurun_out/b_$label.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))" 2>&1 | tail -1)"; }
for n in 8192 65536 1048576 16777216; do
  for lay in 1 2; do ENVS="DSFFT_MP_F16_LAYOUT=$lay" b n${n}_l$lay --n $n; done
done
for st in 1 2 3; do ENVS="DSFFT_MP_STAGES=$st" b n65536_p_s$st --n 65536; done
