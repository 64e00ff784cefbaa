#!/bin/bash
# K13 with the fast-decaying nodes folded into the head (FRAQ_K13_FOLD = max fold levels; 0 = off)
O=gpurun_out/k13fold; mkdir -p $O
for w in C3 C5 C5-SBD C4; do
  for f in 0 16 24 32 48; do
    st=4; [ $w = C4 ] && st=2; [ $w = C3 ] && st=10
    FRAQ_K13_FOLD=$f timeout 600 python bench.py --workload $w --steps $st --no-cpu-baseline > $O/${w}_$f.json 2> $O/${w}_$f.err
    echo "$w fold<=$f rc=$? $(python -c 'import json,sys; d=json.load(open(sys.argv[1])); print("value %.4e e2e %.4e ms %.3f" % (d["value"], d["e2e"]["value"], d["ms_per_step"]))' $O/${w}_$f.json 2>&1 | tail -1)"
  done
done
