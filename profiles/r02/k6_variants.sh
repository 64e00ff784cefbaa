#!/bin/bash
for v in "default" "FRAQ_PHYS_NOGRAPH=1" "FRAQ_K6_NOREFINE=1"; do
  if [ "$v" = default ]; then env_=""; else env_="$v"; fi
  echo "$v: $(env $env_ python profiles/r02/ncu_drivers.py k6split 2>&1 | tail -1)"
done
