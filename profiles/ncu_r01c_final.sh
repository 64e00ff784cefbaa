#!/bin/bash
# Round-1 closing evidence, third session (final tree) (one B200 under gpurun): GPU suite, smoke, C2 bench
# line with CPU baseline, reference arm, ncu launch list of a short bench run (only after the same
# command exited 0 without ncu), and full-size FFPE bench lines.
mkdir -p gpurun_out/final3
O=gpurun_out/final3
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
echo launches=$?
timeout 900 python bench.py --workload C5 --steps 16 > $O/bench_C5_full.json 2> $O/bench_C5_full.err; echo c5=$?
timeout 900 python bench.py --workload C5-SBD --steps 16 > $O/bench_C5SBD_full.json 2> $O/bench_C5SBD_full.err; echo c5sbd=$?
timeout 600 python bench.py --workload C3 > $O/bench_C3.json 2> $O/bench_C3.err; echo c3=$?
timeout 600 python bench.py --workload C4 --steps 5 > $O/bench_C4.json 2> $O/bench_C4.err; echo c4=$?
