#!/bin/bash
# K13: the known part's older rows on the GEMM warps (default) vs all of it on the solver warps
O=gpurun_out/k13split; mkdir -p $O
for w in C5-SBD C4 C5 C3; do
  for v in "X=1" "FRAQ_K13_NOSPLIT=1" "FRAQ_K13_LCAP=80" "FRAQ_K13_LCAP=56"; do
    st=3; [ $w = C4 ] && st=2; [ $w = C3 ] && st=10
    env $v timeout 600 python bench.py --workload $w --steps $st --no-cpu-baseline > $O/${w}_$v.json 2> $O/${w}_$v.err
    echo "$w $v rc=$? $(python -c 'import json,sys; d=json.load(open(sys.argv[1])); print("value %.4e e2e %.4e ms %.3f" % (d["value"], d["e2e"]["value"], d["ms_per_step"]))' $O/${w}_$v.json 2>&1 | tail -1)"
  done
done
