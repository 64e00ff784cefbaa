#!/bin/bash
# e2e with the new default (64-level chunks at C2, ramped) against neighbours
for v in "X=1" "FRAQ_HOST_CHUNK=96" "FRAQ_HOST_CHUNK=32 FRAQ_HOST_NORAMP=1" "FRAQ_HOST_STAGES=3" "X=1"; do
  echo "== $v $(env $v timeout 300 python bench.py --steps 8 --warmup 3 --e2e-steps 8 --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("value %.4e e2e %.4e" % (d["value"], d["e2e"]["value"]))')"
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fir.py tests/test_bench_contract.py tests/test_integration_docs.py -x -q -m gpu 2>&1 | tail -2
