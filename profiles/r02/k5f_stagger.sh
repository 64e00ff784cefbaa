#!/bin/bash
# K5f: odd CTAs window-first / even CTAs state-first, against all CTAs state-first
# (the stagger was measured on a scratch tree: -DFRAQ_K5F_NOSTAGGER is not a switch of the committed kernel)
timeout 600 python -m pytest tests/test_gpu_fir.py -x -q 2>&1 | tail -1
echo "staggered:   $(timeout 200 python profiles/r02/k5f_time.py 2>&1 | grep -E 'K5f')"
echo "staggered:   $(timeout 200 python profiles/r02/k5f_time.py 2>&1 | grep -E 'K5f')"
touch paper_1901_05128_b200/csrc/history_fir.cu
FRAQ_NVCC_FLAGS="-DFRAQ_K5F_NOSTAGGER" python -m paper_1901_05128_b200.build > /dev/null 2>&1
echo "state first: $(timeout 200 python profiles/r02/k5f_time.py 2>&1 | grep -E 'K5f')"
echo "state first: $(timeout 200 python profiles/r02/k5f_time.py 2>&1 | grep -E 'K5f')"
