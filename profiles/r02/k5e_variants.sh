#!/bin/bash
# K5e timing-bound switches (results of the variants are wrong on purpose; only the time counts)
for v in "" "-DFRAQ_EXP_NOREDUCE" "-DFRAQ_EXP_NODMUL" "-DFRAQ_EXP_NOSYNC" "-DFRAQ_EXP_NOFIR" "-DFRAQ_EXP_NOREDUCE -DFRAQ_EXP_NODMUL" "-DFRAQ_EXP_NOREDUCE -DFRAQ_EXP_NODMUL -DFRAQ_EXP_NOSYNC"; do
  touch paper_1901_05128_b200/csrc/history_fir.cu
  FRAQ_NVCC_FLAGS="$v" python -m paper_1901_05128_b200.build > /dev/null 2>&1
  echo "variant [$v] $(timeout 120 python profiles/r02/k5e_time.py 65536 1024 6 | tail -1 | cut -c1-90)"
done
touch paper_1901_05128_b200/csrc/history_fir.cu
python -m paper_1901_05128_b200.build > /dev/null 2>&1
