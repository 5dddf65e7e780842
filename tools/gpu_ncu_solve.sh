mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:solve_tma_kernel -c 1 \
    -o gpurun_out/prof_solve_l0 -f python tools/prof_one.py 65536,64,1 > gpurun_out/ncu_solve.log 2>&1
echo ncu=$?
ncu -i gpurun_out/prof_solve_l0.ncu-rep --page raw --csv > gpurun_out/prof_solve_l0_raw.csv 2>&1
ncu -i gpurun_out/prof_solve_l0.ncu-rep --page details --csv 2>/dev/null | grep -iE "Throughput|Duration|Eligible|Issued|Active Warps|Bandwidth" | head -30
