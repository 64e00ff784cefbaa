#!/bin/bash
# Round-1 ncu evidence (run under gpurun on one B200).  Each ncu pass follows a plain run of the
# same command that exited 0.
set -x
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launches=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:run_kernel -s 3 -c 1 \
    -o gpurun_out/prof_k5b $CMD > gpurun_out/ncu_k5b.log 2>&1
echo k5b=$?
$CMD > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 10 -c 2 \
    -o gpurun_out/prof_k5 $CMD > gpurun_out/ncu_k5.log 2>&1
echo k5=$?
