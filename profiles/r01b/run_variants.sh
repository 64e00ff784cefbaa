#!/bin/bash
# times each built K5d variant twice (interleaved) on one B200
mkdir -p gpurun_out
for rep in 1 2; do
for v in "$@"; do
  timeout 300 python profiles/microbench/time_k5d_var.py gpurun_variants/$v 2>&1 | tail -1
done
done
