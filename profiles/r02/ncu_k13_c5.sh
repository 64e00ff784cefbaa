#!/bin/bash
O=gpurun_out/r02k13c5; mkdir -p $O
for s in FastSBD FastBE; do
python profiles/r02/ncu_drivers.py c5batch $s > $O/plain_$s.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k13_kernel -c 1 \
    -o $O/ncu_k13_$s python profiles/r02/ncu_drivers.py c5batch $s > $O/ncu_$s.log 2>&1; echo $s=$?
done
