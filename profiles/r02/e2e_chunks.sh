#!/bin/bash
# e2e (host buffers through fraq_hist_run) against the host-path chunk height and staging depth
for v in "X=1" "FRAQ_HOST_CHUNK=16" "FRAQ_HOST_CHUNK=64" "FRAQ_HOST_CHUNK=128" "FRAQ_HOST_STAGES=3" "FRAQ_HOST_STAGES=4" "FRAQ_NO_K5E=1"; do
  echo "== $v $(env $v timeout 300 python bench.py --steps 8 --warmup 3 --e2e-steps 4 --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("value %.4e e2e %.4e step_ms %s" % (d["value"], d["e2e"]["value"], d["step_ms_min_max"]))')"
done
