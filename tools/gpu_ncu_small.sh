mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:factor_small_kernel -c 1 \
    -o gpurun_out/prof_small -f python tools/prof_one.py 1048576,8,1 > gpurun_out/ncu_small.log 2>&1
echo ncu=$?
ncu -i gpurun_out/prof_small.ncu-rep --page raw --csv > gpurun_out/prof_small_raw.csv 2>&1
