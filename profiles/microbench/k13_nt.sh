#!/bin/bash
# K13 GEMM-warp width (FRAQ_K13_NT: 8 NT nodes per warp, fewer GEMM warps per SM sub-partition)
# on C5-shaped BE / BDF2 (37 instances, N = 16384) and the C4 loop
export PYTHONUNBUFFERED=1
for rep in 1 2; do
  for e in "" 11; do
    for sc in FastBE FastSBD; do
      echo -n "nt=$e "; FRAQ_K13_NT=$e timeout 300 python profiles/microbench/k13_probe.py $sc 37 16384 2>&1 | tail -1
    done
  done
  for e in "" 9 11; do
    echo -n "nt=$e C4 "; FRAQ_K13_NT=$e timeout 300 python profiles/microbench/c4_drivers.py 8192 transposed 2>&1 | tail -1
  done
done
