# FFPE bench lines (C3, C4, C5, C5-SBD) and K13 DRAM traffic / duration under ncu (after each
# plain run exits 0).
mkdir -p gpurun_out
for w in C3 C4 C5 C5-SBD; do
  python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err || { echo "bench $w failed"; tail -5 gpurun_out/bench_$w.err; continue; }
  tail -1 gpurun_out/bench_$w.json
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:k13_kernel -c 1 --csv python bench.py --workload $w --steps 1 --warmup 0 --no-cpu-baseline \
      > gpurun_out/ncu_k13_$w.csv 2> gpurun_out/ncu_k13_$w.err || echo "ncu $w failed"
done
