#!/bin/bash
# K13 shape variants at C3 (one instance: 256 tasks of 16 modes for 296 CTA slots).
O=gpurun_out/r02k13; mkdir -p $O
for v in "default" "FRAQ_K13_NT=8" "FRAQ_K13_RB1=1"; do
  if [ "$v" = default ]; then env_=""; else env_="$v"; fi
  env $env_ timeout 300 python bench.py --workload C3 --steps 10 --warmup 3 --no-cpu-baseline > $O/c3_${v//=/_}.json 2>&1
  echo "$v $(python -c "import json;d=json.loads(open('$O/c3_${v//=/_}.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['frac'])")"
done
