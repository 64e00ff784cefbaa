#!/bin/bash
# C2 bench value only (no CPU baseline, 1 e2e step), N runs
for r in $(seq 1 ${1:-2}); do
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | \
    python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["e2e"]["value"])'
done
