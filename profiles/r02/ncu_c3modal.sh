#!/bin/bash
O=gpurun_out/r02k13; mkdir -p $O
python profiles/r02/ncu_drivers.py c3modal > $O/c3modal_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c3modal_launches.csv \
    python profiles/r02/ncu_drivers.py c3modal > $O/c3modal_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k13_kernel -c 1 \
    -o $O/ncu_c3_k13 python profiles/r02/ncu_drivers.py c3modal > $O/ncu_c3_k13.log 2>&1; echo k13=$?
