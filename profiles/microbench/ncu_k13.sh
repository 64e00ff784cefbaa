mkdir -p gpurun_out
set -x
python profiles/microbench/k13_probe.py FastBE 4 16384 && \
ncu --set full --import-source on --clock-control none -k regex:k13_kernel -c 1 -o gpurun_out/k13_be -f python profiles/microbench/k13_probe.py FastBE 4 16384 > gpurun_out/ncu_k13_be.log 2>&1
python profiles/microbench/k13_probe.py FastSBD 4 16384 && \
ncu --set full --import-source on --clock-control none -k regex:k13_kernel -c 1 -o gpurun_out/k13_sbd -f python profiles/microbench/k13_probe.py FastSBD 4 16384 > gpurun_out/ncu_k13_sbd.log 2>&1
mkdir -p gpurun_out; ls -la gpurun_out
