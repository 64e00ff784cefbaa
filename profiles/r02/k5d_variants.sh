#!/bin/bash
# K5d instruction-order variants (experiment switches), C2 bench value each.
for v in "" "-DFRAQ_EXP_INTERLEAVE" "-DFRAQ_EXP_INTERLEAVE2"; do
  touch paper_1901_05128_b200/csrc/history_dmma.cu
  FRAQ_NVCC_FLAGS="$v" python -m paper_1901_05128_b200.build > /dev/null 2>&1
  echo "variant [$v] $(bash profiles/r02/c2_value.sh 2 | tr '\n' ' ')"
done
touch paper_1901_05128_b200/csrc/history_dmma.cu
python -m paper_1901_05128_b200.build > /dev/null 2>&1
