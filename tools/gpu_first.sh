#!/bin/bash
# first GPU pass: smoke, parity tests, bench sweep
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_base.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/bench_base.log
for cfg in "2 12" "2 16" "3 8" "4 6" "2 8"; do
  set -- $cfg
  DSFFT_STAGES=$1 DSFFT_GROUPS=$2 timeout 120 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_s$1_g$2.log 2>&1
  echo "S=$1 G=$2: $(python -c "import json,sys; d=json.loads(open('gpurun_out/bench_s$1_g$2.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'])" 2>&1)"
done
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench full rc=$?"
tail -1 gpurun_out/bench_full.log
