#!/bin/bash
# absolute FMA-pipe instruction counts + DRAM bytes for the headline kernels
cd "$GRAFT_REPO_ROOT" || exit 1
M=sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fma_type_fp16.sum,sm__inst_executed_pipe_fp16.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_lsu.sum
for cfg in "fp16 1048576" "fp32 524288"; do
  set -- $cfg
  CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-accuracy --precision $1 --batch $2"
  $CMD > gpurun_out/cnt_plain_$1.log 2>&1 && ncu --metrics $M --clock-control none -k regex:fft_small -s 3 -c 1 --csv --log-file gpurun_out/counters_$1.csv $CMD > gpurun_out/cnt_ncu_$1.log 2>&1
  echo "$1 rc=$?"
done
