mkdir -p gpurun_out
python profiles/microbench/k5d_short.py 8 > gpurun_out/short_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:run3_kernel -s 4 -c 1 \
    -o gpurun_out/prof_k5d_short -f python profiles/microbench/k5d_short.py 8 > gpurun_out/ncu_short.log 2>&1
echo short=$?
