for d in gpurun_variants/*; do python profiles/microbench/time_k5c.py $d 2>&1 | tail -1; done
