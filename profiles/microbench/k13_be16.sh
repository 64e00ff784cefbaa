#!/bin/bash
# BE (J <= 256): 8 GEMM warps of 64 nodes (default, two CTAs per SM) vs 4 of 128 (FRAQ_K13_NT=16)
export PYTHONUNBUFFERED=1
for rep in 1 2; do for e in "" 16; do
  echo -n "nt=$e "; FRAQ_K13_NT=$e timeout 300 python profiles/microbench/k13_probe.py FastBE 37 16384 2>&1 | tail -1
done; done
FRAQ_K13_NT=16 timeout 600 python -m pytest tests/test_gpu_modal.py -m gpu -x -q 2>&1 | tail -2
