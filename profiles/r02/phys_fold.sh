#!/bin/bash
# Physical FFPE stepper with folded kernels in its K5 pass (one B200): parity suites that touch the
# physical path, then C3 / C5 physical bench lines with and without the fold.
O=gpurun_out/s5e; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stepper.py tests/test_gpu_anchor.py tests/test_gpu_configs.py tests/test_gpu_modal.py -x -q -k "ffpe or stepper or anchor or c3 or c5 or physical or block or trajectory" > $O/tests.log 2>&1; echo tests=$?; tail -5 $O/tests.log
for v in fold nofold; do
  if [ $v = nofold ]; then export FRAQ_NO_PHYS_FOLD=1; else unset FRAQ_NO_PHYS_FOLD; fi
  timeout 600 python bench.py --workload C3 --solver physical --steps 3 --warmup 1 --no-cpu-baseline > $O/bench_C3_phys_$v.json 2> $O/bench_C3_phys_$v.err; echo c3p_$v=$?
  timeout 900 python bench.py --workload C5 --solver physical --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_C5_phys_$v.json 2> $O/bench_C5_phys_$v.err; echo c5p_$v=$?
  timeout 900 python bench.py --workload C5-SBD --solver physical --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_C5SBD_phys_$v.json 2> $O/bench_C5SBD_phys_$v.err; echo c5sp_$v=$?
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/s5e/bench_*_phys_*.json")):
    try:
        j = json.load(open(f))
        print(f.split("/")[-1], "%.4e" % j["value"], "ms/step %.1f" % j["ms_per_step"], j.get("roofline", {}).get("frac"))
    except Exception as e:
        print(f, "ERR", e)
PY
