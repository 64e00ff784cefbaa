#!/bin/bash
# Closing ncu evidence on the final tree (K5e with the 128-bit cross-warp reduction): the launch
# list of the bench command (after it exited 0 without ncu) and one --set full capture of K5e.
O=gpurun_out/r02final4; mkdir -p $O
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $O/launches_C2.csv $CMD > $O/ncu_launch.log 2>&1
echo launches=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:run4_kernel --launch-skip 3 -c 1 \
    -o $O/ncu_k5e $CMD > $O/ncu_k5e.log 2>&1; echo ncu_k5e=$?
timeout 600 python bench.py --scaling strong > $O/bench_C2_strong1.json 2> $O/bench_C2_strong1.err; echo strong=$?
timeout 600 python profiles/r02/strong_slices.py > $O/strong_slices.txt 2>&1; echo slices=$?
