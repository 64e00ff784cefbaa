#!/bin/bash
# K13 RB = 1 shapes (C4: J = 408 at N = 8192; C5-SBD probe) for each built variant
export PYTHONUNBUFFERED=1
for v in "$@"; do
  echo "== $v"
  (cd gpurun_variants/$v && timeout 300 python ../../profiles/microbench/c4_drivers.py 8192 transposed 2>&1 | tail -1)
  (cd gpurun_variants/$v && timeout 300 python ../../profiles/microbench/k13_probe.py FastSBD 64 2048 2>&1 | tail -1)
  (cd gpurun_variants/$v && timeout 300 python ../../profiles/microbench/k13_probe.py FastBE 64 2048 2>&1 | tail -1)
done
