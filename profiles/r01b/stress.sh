#!/bin/bash
# repeated K5d runs under short timeouts (a hang shows up as rc=124)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
fails=0
for i in $(seq 1 12); do timeout 60 python profiles/microbench/k5d_stress.py > /dev/null 2>&1 || { echo "stress $i rc=$?"; fails=$((fails+1)); }; done
for i in 1 2 3; do timeout 120 python profiles/microbench/time_k5d_levels.py . 2>&1 | tail -1 || echo "levels rc=$?"; done
for i in 1 2 3; do timeout 120 python profiles/microbench/time_e2e.py 2>&1 | head -1 || echo "e2e rc=$?"; done
echo "stress fails=$fails"
