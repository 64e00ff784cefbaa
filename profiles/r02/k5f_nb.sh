#!/bin/bash
# K5f: loads in flight per thread (node tables staged in shared memory in both)
O=gpurun_out/s5i; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_fir.py -x -q 2>&1 | tail -2
echo "NB=8: $(timeout 200 python profiles/r02/k5f_time.py 2>&1 | grep -E 'K5f|max')"
for nb in 4 6 12; do
touch paper_1901_05128_b200/csrc/history_fir.cu
FRAQ_NVCC_FLAGS="-DFRAQ_K5F_NB=$nb" python -m paper_1901_05128_b200.build > /dev/null 2>&1
echo "NB=$nb: $(timeout 200 python profiles/r02/k5f_time.py 2>&1 | grep -E 'K5f')"
done
