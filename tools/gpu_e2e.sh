#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for c in 16 32 64 128 256; do
  DSFFT_HOST_CHUNK_MB=$c timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-accuracy --e2e-steps 5 > gpurun_out/e2e_$c.log 2>&1
  echo "chunk=$c: $(python -c "import json; d=json.loads(open('gpurun_out/e2e_$c.log').read().strip().splitlines()[-1]); e=d['e2e']; print(round(e['value']/1e6,2),'M/s', round(e['ms_per_step'],2),'ms', round((e['h2d_bytes_per_step']+e['d2h_bytes_per_step'])/e['ms_per_step']/1e6,1),'GB/s total')" 2>&1 | tail -1)"
done
nvidia-smi -q | grep -iA3 "PCIe Generation\|Link Width" | head -12
