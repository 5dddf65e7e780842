#!/bin/bash
# final validation of the round (after the d = 4 solve work): GPU suite, smoke, bench lines
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/h_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/h_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/h_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/h_bench_cfg2.log 2>&1; echo "rc=$?" >> gpurun_out/h_bench_cfg2.log
timeout 1200 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu > gpurun_out/h_bench_cfg5.log 2>&1; echo "rc=$?" >> gpurun_out/h_bench_cfg5.log
BTD_BENCH_GLOO=1 timeout 1500 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/h_bench_cfg5_n2.log 2>&1; echo "rc=$?" >> gpurun_out/h_bench_cfg5_n2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/h_launches_cfg5.csv python tools/prof_dev.py 1048576,64,4 1 > /dev/null 2>&1
