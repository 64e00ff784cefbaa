#!/bin/bash
# K5d state-GEMM instruction-order variants (experiment switches), C2 bench value each.
for v in "" "-DFRAQ_EXP_DMUL_FIRST" "-DFRAQ_EXP_SPLITK"; do
  touch paper_1901_05128_b200/csrc/history_dmma.cu
  FRAQ_NVCC_FLAGS="$v" python -m paper_1901_05128_b200.build > /dev/null 2>&1
  for r in 1 2; do
    echo "variant [$v] $(python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"])')"
  done
done
touch paper_1901_05128_b200/csrc/history_dmma.cu
python -m paper_1901_05128_b200.build > /dev/null 2>&1
