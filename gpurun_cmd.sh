timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 16 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.log 2>&1; echo bench=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench4.log').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['roofline_step_kernel']['frac'], d['e2e']['value'])"
