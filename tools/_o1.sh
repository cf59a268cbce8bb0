cd $GRAFT_REPO_ROOT
DSFFT_MP_FUSED=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -k "65536 or fused or many_chunks or odd_chunks" > gpurun_out/o1.log 2>&1; echo rc=$? >> gpurun_out/o1.log; tail -2 gpurun_out/o1.log
for cfg in "1 1" "1 2" "0 1"; do set -- $cfg; for p in fp16 fp32; do
DSFFT_MP_FUSED=1 DSFFT_MP_OCTET=$1 DSFFT_FUSED_LAG=$2 timeout 120 python bench.py --n 65536 --precision $p --steps 20 --warmup 3 --no-e2e --no-cpu --no-accuracy --sustained-seconds 0 2>&1 | grep '^{' | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('octet=$1 lag=$2 $p', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3))"
done; done
DSFFT_MP_FUSED=1 KREGEX=mp_octet SKIP=3 tools/gpu_ncu.sh "oct16:--n 65536" > /dev/null 2>&1
