#!/bin/bash
# final validation after the d = 1 backward change: GPU suite, smoke, bench cfg2 / cfg5, cfg2 launch list
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -rA --durations=10 > gpurun_out/j_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/j_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/j_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/j_bench_cfg2.log 2>&1; echo "rc=$?" >> gpurun_out/j_bench_cfg2.log
timeout 1200 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu > gpurun_out/j_bench_cfg5.log 2>&1; echo "rc=$?" >> gpurun_out/j_bench_cfg5.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j_launches_cfg2.csv python tools/prof_one.py 65536,64,1 2 > /dev/null 2>&1
