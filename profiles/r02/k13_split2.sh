#!/bin/bash
# K13 with the split known part: head cap sweep
O=gpurun_out/k13split2; mkdir -p $O
for w in C5-SBD C4 C5 C3; do
  for v in 64 72 80 88 96 104; do
    st=3; [ $w = C4 ] && st=2; [ $w = C3 ] && st=10
    FRAQ_K13_LCAP=$v timeout 600 python bench.py --workload $w --steps $st --no-cpu-baseline > $O/${w}_$v.json 2> $O/${w}_$v.err
    echo "$w cap $v rc=$? $(python -c 'import json,sys; d=json.load(open(sys.argv[1])); print("value %.4e e2e %.4e ms %.3f" % (d["value"], d["e2e"]["value"], d["ms_per_step"]))' $O/${w}_$v.json 2>&1 | tail -1)"
  done
done
