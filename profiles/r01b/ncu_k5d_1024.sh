#!/bin/bash
# Session-2: bench line (1024-level steps) and ncu full capture of one 1024-level K5d launch
# (DRAM traffic per launch for bench.py's roofline.traffic).  ncu only after a plain run exits 0.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/b1024.json 2> gpurun_out/b1024.err; echo bench=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain1024.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:run3_kernel -s 3 -c 1 \
    -o gpurun_out/prof_k5d_1024 -f $CMD > gpurun_out/ncu_k5d_1024.log 2>&1
echo k5d=$?
