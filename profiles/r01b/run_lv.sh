#!/bin/bash
# per-call K5d time vs levels and the C2 512-level timing, for each built variant (short timeouts)
export PYTHONUNBUFFERED=1
for v in "$@"; do
  timeout 120 python profiles/microbench/time_k5d_levels.py gpurun_variants/$v 2>&1 | tail -8; echo "rc=$?"
  timeout 120 python profiles/microbench/time_k5d_var.py gpurun_variants/$v 2>&1 | tail -1
done
