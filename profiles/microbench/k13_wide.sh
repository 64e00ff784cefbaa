export PYTHONUNBUFFERED=1
for rep in 1 2; do
for nar in "" 1; do
  echo "== narrow=$nar"
  FRAQ_K13_NARROW=$nar timeout 300 python profiles/microbench/k13_probe.py FastSBD 37 16384 2>&1 | tail -1
  FRAQ_K13_NARROW=$nar timeout 300 python profiles/microbench/c4_drivers.py 8192 transposed 2>&1 | tail -1
done
done
timeout 900 python -m pytest tests/test_gpu_modal.py tests/test_gpu_configs.py -m gpu -x -q 2>&1 | tail -3
