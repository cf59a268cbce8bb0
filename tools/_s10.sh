cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x --timeout 300 -k "multipass or config5 or fused or random" > gpurun_out/s10.log 2>&1; echo rc=$? >> gpurun_out/s10.log; tail -2 gpurun_out/s10.log
for n in 524288 1048576; do for p in fp16 fp32; do for sp in default old; do
if [ $sp = old ]; then if [ $n = 524288 ]; then export DSFFT_MP_SPLIT=7,6,6; else export DSFFT_MP_SPLIT=7,7,6; fi; else unset DSFFT_MP_SPLIT; fi
timeout 120 python bench.py --n $n --precision $p --steps 20 --warmup 3 --no-e2e --no-cpu --no-accuracy --sustained-seconds 0 2>&1 | grep '^{' | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('n=$n $p split=$sp', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3), 'launches', d['roofline']['launches_per_step'])"
done; done; done
