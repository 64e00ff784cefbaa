#!/bin/bash
for st in 2 3 4; do for ch in "" 64; do
  FRAQ_HOST_STAGES=$st FRAQ_HOST_CHUNK=$ch timeout 300 python profiles/microbench/e2e_stages.py 2>&1 | tail -1
done; done
