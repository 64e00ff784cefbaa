#!/bin/bash
# Round-2 closing evidence for the FFPE configurations with the K13 head fold (one B200):
# every FFPE bench line and ncu captures of K13 at C5 shape (BDF2 and BE).
O=gpurun_out/r02final3; mkdir -p $O
timeout 600 python bench.py --workload C3 > $O/bench_C3.json 2> $O/bench_C3.err; echo c3=$?
timeout 900 python bench.py --workload C4 --steps 3 > $O/bench_C4.json 2> $O/bench_C4.err; echo c4=$?
timeout 900 python bench.py --workload C5 --steps 4 > $O/bench_C5.json 2> $O/bench_C5.err; echo c5=$?
timeout 900 python bench.py --workload C5-SBD --steps 4 > $O/bench_C5SBD.json 2> $O/bench_C5SBD.err; echo c5sbd=$?
for s in FastSBD FastBE; do
python profiles/r02/ncu_drivers.py c5batch $s > $O/plain_$s.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k13_kernel -c 1 \
    -o $O/ncu_k13_$s python profiles/r02/ncu_drivers.py c5batch $s > $O/ncu_$s.log 2>&1; echo $s=$?
done
