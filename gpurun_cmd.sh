timeout 900 python bench.py --steps 8 > gpurun_out/bench_cpu.log 2>gpurun_out/bench_cpu.err; echo bench=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_cpu.log').read().strip().splitlines()[-1]); print(d['value'], d['cpu_baseline'])"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?; tail -1 gpurun_out/bench_ref.log | cut -c1-300
