#!/bin/bash
# K13 RB = 2 shapes at the full C5 horizon (FastBE, J <= 256) for each built variant, twice
export PYTHONUNBUFFERED=1
for rep in 1 2; do
for v in "$@"; do
  echo -n "$v "; (cd gpurun_variants/$v && timeout 300 python ../../profiles/microbench/k13_probe.py FastBE 64 16384 2>&1 | tail -1)
done
done
