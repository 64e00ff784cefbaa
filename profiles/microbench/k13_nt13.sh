#!/bin/bash
# wide K13: 104-node GEMM warps (FRAQ_K13_NT=13: 5 per field, 12 warps, 168 registers) vs the
# default 72 / 88-node warps, on C4 and C5-shaped BDF2
export PYTHONUNBUFFERED=1
for rep in 1 2; do for e in "" 13 16; do
  echo -n "nt=$e "; FRAQ_K13_NT=$e timeout 300 python profiles/microbench/k13_probe.py FastSBD 37 16384 2>&1 | tail -1
  echo -n "nt=$e C4 "; FRAQ_K13_NT=$e timeout 300 python profiles/microbench/c4_drivers.py 8192 transposed 2>&1 | tail -1
done; done
FRAQ_K13_NT=16 timeout 600 python -m pytest tests/test_gpu_modal.py -m gpu -x -q -k "wide or 2d" 2>&1 | tail -2
