#!/bin/bash
# K5f: where do the window rows come from?  Default vs the input ring as a persisting L2 window.
O=gpurun_out/s5h; mkdir -p $O
echo "default:        $(timeout 200 python profiles/r02/k5f_time.py 2>&1 | grep K5f)"
# (the FRAQ_K5F_L2PERSIST switch existed on the tree of commit 6e10ee6 only)
echo "L2 persisting:  $(FRAQ_K5F_L2PERSIST=1 timeout 200 python profiles/r02/k5f_time.py 2>&1 | grep -E 'K5f|rror' | head -3)"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:step_fir_kernel --launch-skip 100 -c 1 \
    -o $O/ncu_k5f python profiles/r02/k5f_time.py > $O/ncu_k5f.log 2>&1; echo ncu_k5f=$?
FRAQ_K5F_L2PERSIST=1 timeout 600 ncu --set full --clock-control none -k regex:step_fir_kernel --launch-skip 100 -c 1 \
    -o $O/ncu_k5f_persist python profiles/r02/k5f_time.py > $O/ncu_k5f_persist.log 2>&1; echo ncu_k5f_persist=$?
