#!/bin/bash
# Round-2 measurements (one B200 under gpurun): C2 headline + reference arm, FFPE lines (modal and
# physical C3), ncu of the physical kernels (K5 FFPE mode, K6) and of the C4 DST GEMM (K12).
O=gpurun_out/r02m1
mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_C2.json 2> $O/bench_C2.err; echo c2=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_C2_ref.json 2> $O/bench_C2_ref.err; echo ref=$?
timeout 900 python bench.py --workload C3 --solver physical --steps 2 --warmup 1 > $O/bench_C3_phys.json 2> $O/bench_C3_phys.err; echo c3p=$?
timeout 600 python bench.py --workload C3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err; echo c3=$?
python profiles/r02/ncu_drivers.py c3phys 64 > $O/c3phys_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"solve_kernel|step_kernel" --launch-skip 20 -c 2 \
    -o $O/ncu_c3phys python profiles/r02/ncu_drivers.py c3phys 64 > $O/ncu_c3phys.log 2>&1; echo ncu_c3phys=$?
python profiles/r02/ncu_drivers.py c4dst > $O/c4dst_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dst_kernel --launch-skip 1 -c 1 \
    -o $O/ncu_c4dst python profiles/r02/ncu_drivers.py c4dst > $O/ncu_c4dst.log 2>&1; echo ncu_c4dst=$?
