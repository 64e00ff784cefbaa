#!/bin/bash
# Third-session K13 evidence: warp-slot probe (solver warps' SM sub-partitions with 2 CTAs/SM),
# K13 timing on a full-wave C5-shaped batch (37 instances x 256 tasks = 32 waves of 296 CTAs),
# then one ncu --set full capture per scheme (after the plain run exited 0).
mkdir -p gpurun_out/k13
O=gpurun_out/k13
./profiles/microbench/mb_warpslot > $O/warpslot.txt 2>&1; echo slot=$?
for sc in FastBE FastSBD; do
  timeout 300 python profiles/microbench/k13_probe.py $sc 37 4096 > $O/time_$sc.txt 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k13_kernel -c 1 \
      -o $O/k13_$sc -f python profiles/microbench/k13_probe.py $sc 37 4096 > $O/ncu_$sc.log 2>&1
  echo $sc=$?
done
