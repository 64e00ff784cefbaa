#!/bin/bash
# ncu --set full of K13 (one launch, C5-shaped 37 instances x 4096 levels) for built variants
mkdir -p gpurun_out/k13v
for v in "$@"; do
  for sc in FastSBD FastBE; do
    (cd gpurun_variants/$v && timeout 300 python ../../profiles/microbench/k13_probe.py $sc 37 4096 > /dev/null 2>&1 && \
     timeout 600 ncu --set full --import-source on --clock-control none -k regex:k13_kernel -c 1 \
       -o ../../gpurun_out/k13v/${v}_$sc -f python ../../profiles/microbench/k13_probe.py $sc 37 4096 > ../../gpurun_out/k13v/${v}_$sc.log 2>&1)
    echo $v $sc $?
  done
done
