timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
python profiles/microbench/time_k5c.py .
FRAQ_K5C=1 python profiles/microbench/time_k5c.py .
