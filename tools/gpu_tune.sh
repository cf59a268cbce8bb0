#!/bin/bash
# Launch-shape / layout sweep for one workload (run under gpurun).
#
#   N=1024 PREC=fp16 tools/gpu_tune.sh "DSFFT_STAGES=2 DSFFT_GROUPS=12" "DSFFT_STAGES=3" ...
#
# Each argument is a set of environment overrides for one bench run.  Knobs:
#   single kernel (N <= 4096)
#     DSFFT_STAGES        item buffers per group (ring depth)
#     DSFFT_GROUPS        independent thread groups per CTA
#     DSFFT_F16_LAYOUT    1 = transform pairs, 2 = one complex per f16x2 register
#     DSFFT_CTAS_PER_SM   persistent CTAs per SM
#   multipass (N >= 8192)
#     DSFFT_MP_STAGES     ring depth;  DSFFT_MP_GROUPS  tile groups per CTA
#     DSFFT_MP_CHUNK_MB   batch chunk per launch sequence
#     DSFFT_MP_F16_LAYOUT 1 = transform pairs, 2 = one complex per register
#     DSFFT_MP_SPLIT      pass-group sizes, e.g. "9,7" (each 6..9, summing to log2 N)
#   host pipeline
#     DSFFT_HOST_CHUNK_MB chunk of dsfft_execute_host's H2D/kernel/D2H pipeline
#   A/B builds
#     DSFFT_LIBRARY       path of another libdsfft.so build to load instead
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
N=${N:-1024}
PREC=${PREC:-fp16}
i=0
for envs in "$@"; do
  i=$((i + 1))
  env $envs timeout 300 python bench.py --n "$N" --precision "$PREC" --steps "${STEPS:-30}" \
      --warmup 3 --no-cpu --no-e2e --no-accuracy > "gpurun_out/tune_$i.log" 2>&1
  echo "[$envs] $(python -c "import json; d=json.loads(open('gpurun_out/tune_$i.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'], 4), 'ms', round(d['roofline']['frac'], 4), 'of HBM')" 2>&1 | tail -1)"
done
