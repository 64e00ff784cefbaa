#!/bin/bash
# Final-tree FFPE lines (modal default) + physical C3, one B200.
O=gpurun_out/r02final5; mkdir -p $O
timeout 600 python bench.py --workload C3 > $O/bench_C3.json 2> $O/bench_C3.err; echo c3=$?
timeout 900 python bench.py --workload C4 --steps 3 > $O/bench_C4.json 2> $O/bench_C4.err; echo c4=$?
timeout 900 python bench.py --workload C5 --steps 4 > $O/bench_C5.json 2> $O/bench_C5.err; echo c5=$?
timeout 900 python bench.py --workload C5-SBD --steps 4 > $O/bench_C5SBD.json 2> $O/bench_C5SBD.err; echo c5sbd=$?
timeout 900 python bench.py --workload C3 --solver physical --steps 3 --warmup 1 > $O/bench_C3_phys.json 2> $O/bench_C3_phys.err; echo c3p=$?
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_C2_20.json 2> $O/bench_C2_20.err; echo c2=$?
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r02final5/bench_*.json")):
    try:
        j = json.load(open(f))
        print(f.split("/")[-1], "%.4e" % j["value"], "ms/step %.3f" % j["ms_per_step"], "e2e %.3e" % j["e2e"]["value"], "cpu", j.get("cpu_baseline", {}).get("value"))
    except Exception as e:
        print(f, "ERR", e)
PY
