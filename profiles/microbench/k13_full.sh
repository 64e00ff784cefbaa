#!/bin/bash
# K13 timing at full-horizon C5 shapes (37 instances = whole waves, N = 16384) per built variant
export PYTHONUNBUFFERED=1
for rep in 1 2; do
for v in "$@"; do
  for sc in FastBE FastSBD; do
    echo -n "$v "; (cd gpurun_variants/$v && timeout 300 python ../../profiles/microbench/k13_probe.py $sc 37 16384 2>&1 | tail -1)
  done
done
done
