#!/bin/bash
# round-2 bench lines (all BASELINE single-GPU configs), launch lists and ncu --set full captures
mkdir -p gpurun_out
for c in cfg2 cfg1 cfg3 cfg4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/g_bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/g_bench_$c.log
done
for c in 65536,64,1 1048576,8,1; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_launches_$c.csv python tools/prof_one.py $c 2 > /dev/null 2>&1
done
cap() {  # name regex cfg [skip]
  ncu --set full --clock-control none --import-source on -k regex:$2 -s ${4:-0} -c 1 -o gpurun_out/g_ncu_$1 -f python tools/prof_one.py $3 > gpurun_out/g_ncu_$1.log 2>&1
  ncu -i gpurun_out/g_ncu_$1.ncu-rep --page raw --csv > gpurun_out/g_ncu_$1_raw.csv 2>&1
}
cap cfg2_factor_l0 factor_level_kernel 65536,64,1
cap cfg3_factor_l0 factor_small_kernel 1048576,8,1
cap cfg3_solve_l0 solve_small_kernel 1048576,8,1
