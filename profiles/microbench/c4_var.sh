#!/bin/bash
# C4 K13 loop (transposed driver, N = 8192) per built variant
export PYTHONUNBUFFERED=1
for rep in 1 2; do
for v in "$@"; do
  echo -n "$v "; (cd gpurun_variants/$v && timeout 300 python ../../profiles/microbench/c4_drivers.py 8192 transposed 2>&1 | tail -1)
done
done
