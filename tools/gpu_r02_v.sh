#!/bin/bash
# bench lines + launch lists + ncu of the level-0 kernels after the sub-partition roles
mkdir -p gpurun_out
for c in cfg2 cfg1 cfg3 cfg4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/v_bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/v_bench_$c.log
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v_launches_cfg2.csv python tools/prof_one.py 65536,64,1 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:factor_level_kernel -c 1 -o gpurun_out/v_ncu_cfg2_factor_l0 -f python tools/prof_one.py 65536,64,1 > gpurun_out/v_ncu.log 2>&1
ncu -i gpurun_out/v_ncu_cfg2_factor_l0.ncu-rep --page raw --csv > gpurun_out/v_ncu_cfg2_factor_l0_raw.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:factor_small_kernel -c 1 -o gpurun_out/v_ncu_cfg3_factor_l0 -f python tools/prof_one.py 1048576,8,1 >> gpurun_out/v_ncu.log 2>&1
ncu -i gpurun_out/v_ncu_cfg3_factor_l0.ncu-rep --page raw --csv > gpurun_out/v_ncu_cfg3_factor_l0_raw.csv 2>&1
