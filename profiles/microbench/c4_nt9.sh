#!/bin/bash
# C4 K13 loop with 64-node (default) vs 72-node GEMM warps (FRAQ_K13_NT9: 6 warps per field for
# J = 408, 432 padded nodes instead of 448), plus the K13-vs-K11 check under the switch
export PYTHONUNBUFFERED=1
for rep in 1 2; do for e in "" 1; do
  echo -n "nt9=$e "; FRAQ_K13_NT9=$e timeout 300 python profiles/microbench/c4_drivers.py 8192 transposed 2>&1 | tail -1
done; done
FRAQ_K13_NT9=1 timeout 600 python -m pytest tests/test_gpu_modal.py -m gpu -x -q -k "wide or 2d" 2>&1 | tail -2
