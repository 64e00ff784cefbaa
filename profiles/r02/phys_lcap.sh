#!/bin/bash
# Head cap of the folded kernels in the physical stepper (one B200): C5 physical lines.
O=gpurun_out/s5f; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_fir.py -x -q > $O/tests_fir.log 2>&1; echo fir=$?; tail -3 $O/tests_fir.log
for cap in 128 160; do
  export FRAQ_PHYS_LCAP=$cap
  timeout 900 python bench.py --workload C5 --solver physical --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_C5_phys_cap$cap.json 2> $O/bench_C5_phys_cap$cap.err; echo c5p_$cap=$?
  timeout 900 python bench.py --workload C5-SBD --solver physical --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_C5SBD_phys_cap$cap.json 2> $O/bench_C5SBD_phys_cap$cap.err; echo c5sp_$cap=$?
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/s5f/bench_*.json")):
    try:
        j = json.load(open(f))
        print(f.split("/")[-1], "%.4e" % j["value"], "ms/step %.1f" % j["ms_per_step"])
    except Exception as e:
        print(f, "ERR", e)
PY
