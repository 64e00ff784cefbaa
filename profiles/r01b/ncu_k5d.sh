#!/bin/bash
# Session-2 K5d capture: full set with source (stall attribution per SASS line).
mkdir -p gpurun_out
CMD="python profiles/microbench/time_k5c.py ."
$CMD > gpurun_out/k5d_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:run3_kernel -s 2 -c 1 \
    -o gpurun_out/prof_k5d_s2 -f $CMD > gpurun_out/ncu_k5d_s2.log 2>&1
echo k5d=$?
