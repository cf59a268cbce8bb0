#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
C1="python bench.py --n 65536 --steps 1 --warmup 3 --no-cpu --no-e2e"
$C1 > gpurun_out/mp_plain1.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:mp_kernel -s 6 -c 2 -o gpurun_out/prof_mp65536b $C1 > gpurun_out/ncu_mp1.log 2>&1; echo rc1=$?
