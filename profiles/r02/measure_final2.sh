#!/bin/bash
# Round-2 closing evidence for K5e on one B200 (gpurun): the C2 bench line, the reference arm, the
# launch list of the bench command (after it exited 0 without ncu) and an ncu capture of K5e.
O=gpurun_out/r02final2; mkdir -p $O
timeout 900 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err; echo c2=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_C2_ref.json 2> $O/bench_C2_ref.err; echo ref=$?
timeout 900 python bench.py --scaling strong > $O/bench_C2_strong1.json 2> $O/bench_C2_strong1.err; echo strong=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $O/launches_C2.csv $CMD > $O/ncu_launch.log 2>&1
echo launches=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:run4_kernel --launch-skip 3 -c 1 \
    -o $O/ncu_k5e $CMD > $O/ncu_k5e.log 2>&1; echo ncu_k5e=$?
