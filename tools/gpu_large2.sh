#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "multipass" > gpurun_out/pytest_mp.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_mp.log
for n in ${NS:-8192 65536 1048576 16777216}; do
 for p in fp16 fp32; do
  timeout 300 python bench.py --n $n --precision $p --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/large_${n}_$p.log 2>&1
  echo "n=$n $p: $(python -c "import json; d=json.loads(open('gpurun_out/large_${n}_$p.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), d['config']['batch_per_gpu'], round(d['roofline']['frac'],4), d['gpu_launches'])" 2>&1 | tail -1)"
 done
done
