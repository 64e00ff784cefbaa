#!/bin/bash
# Round-2 evidence on one B200 (gpurun): every bench line, the reference arm, the launch list of
# the default bench command (after it exited 0 without ncu) and ncu captures of the top kernels.
O=gpurun_out/r02final; mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_C2.json 2> $O/bench_C2.err; echo c2=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_C2_ref.json 2> $O/bench_C2_ref.err; echo ref=$?
timeout 600 python bench.py --workload C3 > $O/bench_C3.json 2> $O/bench_C3.err; echo c3=$?
timeout 900 python bench.py --workload C3 --solver physical --steps 3 --warmup 1 > $O/bench_C3_phys.json 2> $O/bench_C3_phys.err; echo c3p=$?
timeout 900 python bench.py --workload C4 --steps 3 > $O/bench_C4.json 2> $O/bench_C4.err; echo c4=$?
timeout 900 python bench.py --workload C5 --steps 4 > $O/bench_C5.json 2> $O/bench_C5.err; echo c5=$?
timeout 900 python bench.py --workload C5-SBD --steps 4 > $O/bench_C5SBD.json 2> $O/bench_C5SBD.err; echo c5sbd=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $O/launches_C2.csv $CMD > $O/ncu_launch.log 2>&1
echo launches=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:run3_kernel --launch-skip 3 -c 1 \
    -o $O/ncu_k5d $CMD > $O/ncu_k5d.log 2>&1; echo ncu_k5d=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dst_kernel --launch-skip 1 -c 1 \
    -o $O/ncu_dst python profiles/r02/ncu_drivers.py c4dst > $O/ncu_dst.log 2>&1; echo ncu_dst=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:solve_kernel --launch-skip 100 -c 1 \
    -o $O/ncu_k6 python profiles/r02/ncu_drivers.py c3phys 256 > $O/ncu_k6.log 2>&1; echo ncu_k6=$?
