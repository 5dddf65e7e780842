#!/bin/bash
# full validation + bench lines of the current build (round-2 final)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/x2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/x2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/x2_smoke.log 2>&1
for c in cfg2 cfg1 cfg3 cfg4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/x2_bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/x2_bench_$c.log
done
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu > gpurun_out/x2_bench_cfg5.log 2>&1; echo "rc=$?" >> gpurun_out/x2_bench_cfg5.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/x2_launches_cfg2.csv python tools/prof_one.py 65536,64,1 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:factor_level_kernel -c 1 -o gpurun_out/x2_ncu_cfg2_factor_l0 -f python tools/prof_one.py 65536,64,1 > gpurun_out/x2_ncu.log 2>&1
