#!/bin/bash
# K5e: FIR window length / staged chunk height sweep at C2 (one B200).
# TC = levels per TMA chunk (32: windows up to 72 rows in the 128-row ring; 16: up to 104 rows).
T="timeout 120 python profiles/r02/k5e_time.py 65536 1024 6"
line() { tail -1 | cut -c1-95; }
echo "TC=32 planner      $($T | line)"
for m in 56 64 72; do echo "TC=32 M=$m (ring 256) $(FRAQ_K5E_M=$m $T | line)"; done
touch paper_1901_05128_b200/csrc/history_fir.cu
FRAQ_NVCC_FLAGS="-DFRAQ_K5E_TC=16" python -m paper_1901_05128_b200.build > /dev/null 2>&1
echo "TC=16 planner      $(FRAQ_K5E_DEBUG=1 $T 2>&1 | grep -E 'K5e group 0|DOFs' | cut -c1-120 | tr '\n' ' ')"
for m in 48 56 64 72 80; do echo "TC=16 M=$m          $(FRAQ_K5E_M=$m $T | line)"; done
for w in 3 5; do echo "TC=16 planner NWG=$w $(FRAQ_K5E_NWG=$w $T | line)"; done
touch paper_1901_05128_b200/csrc/history_fir.cu
python -m paper_1901_05128_b200.build > /dev/null 2>&1
