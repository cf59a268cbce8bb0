#!/bin/bash
# ncu evidence for the headline kernel: launch list + one --set full capture
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CMD16="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-accuracy --sustained-seconds 0"
CMD32="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-accuracy --sustained-seconds 0 --precision fp32 --global-batch 524288"
$CMD16 > gpurun_out/plain16.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fp16.csv $CMD16 > gpurun_out/ncu_launch16.log 2>&1
echo "launch list rc=$?"
$CMD16 > gpurun_out/plain16b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fft_small -s 3 -c 1 -o gpurun_out/prof_n1024_fp16 $CMD16 > gpurun_out/ncu_full16.log 2>&1
echo "full16 rc=$?"
$CMD32 > gpurun_out/plain32.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fft_small -s 3 -c 1 -o gpurun_out/prof_n1024_fp32 $CMD32 > gpurun_out/ncu_full32.log 2>&1
echo "full32 rc=$?"
tail -1 gpurun_out/plain16.log; tail -1 gpurun_out/plain32.log
