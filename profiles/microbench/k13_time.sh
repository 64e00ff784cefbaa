#!/bin/bash
# K13 timing on C5-shaped batches (64 instances, 2048 levels, BE and SBD) for each built variant
export PYTHONUNBUFFERED=1
for rep in 1 2; do
for v in "$@"; do
  for sc in FastBE FastSBD; do
    echo -n "$v "; (cd gpurun_variants/$v && timeout 300 python ../../profiles/microbench/k13_probe.py $sc 64 2048 2>&1 | tail -1)
  done
done
done
