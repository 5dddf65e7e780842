# ncu --set full of the level-0 solve pass (solve_tma_kernel) with source-level stall sampling
mkdir -p gpurun_out
CFG=${1:-65536,64,1}
ncu --set full --clock-control none --import-source on -k regex:solve_tma_kernel -c 1 \
    -o gpurun_out/prof_solve_src -f python tools/prof_dev.py $CFG 1 > gpurun_out/ncu_solve_src.log 2>&1
echo ncu=$?
ncu -i gpurun_out/prof_solve_src.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_solve_src_sass.csv 2>&1
ncu -i gpurun_out/prof_solve_src.ncu-rep --page raw --csv > gpurun_out/prof_solve_src_raw.csv 2>&1
