#!/bin/bash
# Closing ncu evidence on the final tree: launch list of the bench command (after it exited 0
# without ncu), --set full captures of K5e (run4_kernel) and K5f (step_fir_kernel).
O=gpurun_out/r02final6; mkdir -p $O
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $O/launches_C2.csv $CMD > $O/ncu_launch.log 2>&1
echo launches=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:run4_kernel --launch-skip 3 -c 1 \
    -o $O/ncu_k5e $CMD > $O/ncu_k5e.log 2>&1; echo ncu_k5e=$?
timeout 600 ncu --set full --import-source on --clock-control none --cache-control none -k regex:step_fir_kernel --launch-skip 100 -c 1 \
    -o $O/ncu_k5f python profiles/r02/k5f_time.py > $O/ncu_k5f.log 2>&1; echo ncu_k5f=$?
