cd "$GRAFT_REPO_ROOT"
for p in fp16 fp32; do
N=524288 PREC=$p STEPS=30 tools/gpu_tune.sh X=1 DSFFT_MP_SPLIT=6,7,6 DSFFT_MP_SPLIT=6,6,7 | sed "s/^/19 $p /"
N=1048576 PREC=$p STEPS=30 tools/gpu_tune.sh X=1 DSFFT_MP_SPLIT=8,6,6 DSFFT_MP_SPLIT=6,7,7 DSFFT_MP_SPLIT=7,6,7 | sed "s/^/20 $p /"
N=2097152 PREC=$p STEPS=30 tools/gpu_tune.sh X=1 DSFFT_MP_SPLIT=8,7,6 DSFFT_MP_SPLIT=9,6,6 DSFFT_MP_SPLIT=6,7,8 | sed "s/^/21 $p /"
N=4194304 PREC=$p STEPS=30 tools/gpu_tune.sh X=1 DSFFT_MP_SPLIT=8,8,6 DSFFT_MP_SPLIT=9,7,6 DSFFT_MP_SPLIT=6,8,8 | sed "s/^/22 $p /"
N=8388608 PREC=$p STEPS=30 tools/gpu_tune.sh X=1 DSFFT_MP_SPLIT=9,8,6 DSFFT_MP_SPLIT=9,7,7 DSFFT_MP_SPLIT=7,8,8 | sed "s/^/23 $p /"
N=16777216 PREC=$p STEPS=30 tools/gpu_tune.sh X=1 DSFFT_MP_SPLIT=9,9,6 DSFFT_MP_SPLIT=9,8,7 DSFFT_MP_SPLIT=6,9,9 | sed "s/^/24 $p /"
done
