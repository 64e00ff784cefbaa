#!/bin/bash
# ncu --set full of the final K13 shapes (C5-shaped: 37 instances, N = 16384): BE (128-node GEMM
# warps, two CTAs per SM) and BDF2 (128-node warps, wide CTA), after plain runs exited 0
mkdir -p gpurun_out/k13v4
O=gpurun_out/k13v4
for sc in FastBE FastSBD; do
  timeout 300 python profiles/microbench/k13_probe.py $sc 37 16384 > $O/probe_$sc.txt 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k13_kernel -c 1 \
      -o $O/k13_$sc -f python profiles/microbench/k13_probe.py $sc 37 16384 > $O/ncu_$sc.log 2>&1
  echo ncu_$sc=$?
done
