#!/bin/bash
# Round-1 closing evidence (one B200, under gpurun): bench lines (C2 default with CPU baseline,
# reference arm), smoke, and ncu (launch list + full captures of K5d and K13).  Every ncu pass
# follows a plain run of the same command that exited 0.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches_final.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launches=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:run3_kernel -s 3 -c 1 \
    -o gpurun_out/prof_k5d_final -f $CMD > gpurun_out/ncu_k5d.log 2>&1
echo k5d=$?
P="python profiles/microbench/k13_probe.py FastBE 4 16384"
$P > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k13_kernel -c 1 \
    -o gpurun_out/prof_k13_final -f $P > gpurun_out/ncu_k13.log 2>&1
echo k13=$?
