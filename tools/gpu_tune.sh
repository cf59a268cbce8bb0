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
#     DSFFT_MP_SPLIT      pass-group sizes, e.g. "9,7" (each 6..10, summing to log2 N)
#     DSFFT_MP_FUSED      1 / 0: force the one-launch (L2-resident) path on / off
#                         (N = 2^14, 2^16, 2^18; default on for fp16 2^14 / 2^16
#                         and fp32 2^14, 6-FMA variants)
#     DSFFT_FUSED_LAG / DSFFT_FUSED_SLOTS / DSFFT_FUSED_TEAMS / DSFFT_FUSED_GROUPS /
#     DSFFT_FUSED_SMS     one-launch lag (units), ring slots, teams, tile groups, SM cap
#     DSFFT_MP_CW=16      16-column tiles in every group from s = 7;
#     DSFFT_MP_CWMASK     ... in the groups of this bit mask only
#     DSFFT_MP_CW10MASK   s = 10 groups of this bit mask on 8-column tiles
#                         (default: the fp32 first group)
#     DSFFT_MP_KEEP       1 / 0: load tiles evict_normal / evict_first (default:
#                         evict_normal only for first-group rows < 128 B)
#     DSFFT_MP_PREFETCH   1 / 0: L2-prefetch the next tile in every group / none;
#     DSFFT_MP_PFMASK     ... in the groups of this bit mask (default: later
#                         groups with s = 9, or s = 10 for fp16 pairs)
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
