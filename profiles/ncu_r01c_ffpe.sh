#!/bin/bash
# Third-session evidence after the K13 changes (wide CTA, GEMM-side partial reduction, folded
# solver coefficients): GPU suite, smoke, full FFPE bench lines, one ncu --set full of K13 per
# scheme (C5-shaped, after the plain run exited 0).
mkdir -p gpurun_out/ffpe3
O=gpurun_out/ffpe3
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --workload C5 --steps 16 > $O/bench_C5_full.json 2> $O/c5.err; echo c5=$?
timeout 900 python bench.py --workload C5-SBD --steps 16 > $O/bench_C5SBD_full.json 2> $O/c5sbd.err; echo c5sbd=$?
timeout 600 python bench.py --workload C4 > $O/bench_C4.json 2> $O/c4.err; echo c4=$?
timeout 600 python bench.py --workload C3 > $O/bench_C3.json 2> $O/c3.err; echo c3=$?
for sc in FastBE FastSBD; do
  timeout 300 python profiles/microbench/k13_probe.py $sc 37 16384 > $O/probe_$sc.txt 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k13_kernel -c 1 \
      -o $O/k13_$sc -f python profiles/microbench/k13_probe.py $sc 37 16384 > $O/ncu_$sc.log 2>&1
  echo ncu_$sc=$?
done
