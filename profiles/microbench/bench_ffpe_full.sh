# Full-size FFPE bench lines: C5 as the complete 4096-instance sweep (16 steps x 256 instances, both
# schemes), C3 and C4 defaults.
mkdir -p gpurun_out
python bench.py --workload C5 --steps 16 > gpurun_out/bench_C5_full.json 2> gpurun_out/bench_C5_full.err; echo c5=$?
python bench.py --workload C5-SBD --steps 16 > gpurun_out/bench_C5SBD_full.json 2> gpurun_out/bench_C5SBD_full.err; echo c5sbd=$?
python bench.py --workload C3 > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo c3=$?
python bench.py --workload C4 > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo c4=$?
