timeout 900 python bench.py > gpurun_out/bench_r01.log 2>gpurun_out/bench_r01.err; echo bench=$?; tail -1 gpurun_out/bench_r01.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:run3_kernel -s 3 -c 1 -o gpurun_out/prof_k5d_r01 $CMD > gpurun_out/ncu_k5d.log 2>&1; echo k5d=$?
$CMD > gpurun_out/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 10 -c 1 -o gpurun_out/prof_k5_r01 $CMD > gpurun_out/ncu_k5.log 2>&1; echo k5=$?
