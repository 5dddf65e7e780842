# one ncu --set full capture of the level-0 factor kernel + the cfg4 bench line
mkdir -p gpurun_out
CFG=${1:-65536,64,1}
ncu --set full --clock-control none --import-source on -k regex:factor_level_kernel -c 1 \
    -o gpurun_out/prof_factor_l0 -f python tools/prof_one.py $CFG > gpurun_out/ncu_full.log 2>&1
echo ncu=$?
ncu -i gpurun_out/prof_factor_l0.ncu-rep --page raw --csv > gpurun_out/prof_factor_l0_raw.csv 2>&1
timeout 900 python bench.py --no-cpu --config cfg4 > gpurun_out/bench_cfg4.log 2>&1; echo cfg4=$?; tail -1 gpurun_out/bench_cfg4.log
