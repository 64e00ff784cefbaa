#!/bin/bash
# K13 head fold with the intermediate tile shapes: default vs no intermediate shapes vs no fold
O=gpurun_out/k13fold2; mkdir -p $O
for w in C3 C5 C5-SBD C4; do
  for v in "X=1" "FRAQ_K13_NOMID=1" "FRAQ_K13_FOLD=0" "FRAQ_K13_FOLD=32" "FRAQ_K13_FOLD=24"; do
    st=4; [ $w = C4 ] && st=2; [ $w = C3 ] && st=10
    env $v timeout 600 python bench.py --workload $w --steps $st --no-cpu-baseline > $O/${w}_$v.json 2> $O/${w}_$v.err
    echo "$w $v rc=$? $(python -c 'import json,sys; d=json.load(open(sys.argv[1])); print("value %.4e e2e %.4e ms %.3f" % (d["value"], d["e2e"]["value"], d["ms_per_step"]))' $O/${w}_$v.json 2>&1 | tail -1)"
  done
done
