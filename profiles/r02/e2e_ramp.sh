#!/bin/bash
# e2e (host buffers through fraq_hist_run): ramped chunk schedule against the uniform one
timeout 900 python -m pytest tests/test_gpu_fir.py tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "not c3_full and not all_lanes and not c5" 2>&1 | tail -2
for v in "FRAQ_HOST_NORAMP=1" "X=1" "FRAQ_HOST_CHUNK=64" "FRAQ_HOST_CHUNK=64 FRAQ_HOST_NORAMP=1" "FRAQ_HOST_CHUNK=128" "FRAQ_HOST_NORAMP=1" "X=1"; do
  echo "== $v $(env $v timeout 300 python bench.py --steps 8 --warmup 3 --e2e-steps 8 --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("value %.4e e2e %.4e" % (d["value"], d["e2e"]["value"]))')"
done
