#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "bit_exact_vs_reference and (2048 or 4096)" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt.log
DSFFT_F16_LAYOUT=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "bit_exact_vs_reference and (2048 or 4096) and fp16" > gpurun_out/pt2.log 2>&1; echo "pytest f16c rc=$?"; tail -1 gpurun_out/pt2.log
b() { local label=$1; shift
  env $ENVS timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-accuracy "$@" > gpurun_out/b_$label.log 2>&1
  echo "$label $ENVS: $(python -c "import json; d=json.loads(open('gpurun_out/b_$label.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))" 2>&1 | tail -1)"; }
for n in 2048 4096; do for st in 1 2; do ENVS="DSFFT_F16_LAYOUT=2 DSFFT_STAGES=$st" b n${n}_c_s$st --n $n; done; done
