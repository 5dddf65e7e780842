#!/bin/bash
# full validation + bench lines of the current build
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -n 1 -p no:cacheprovider > gpurun_out/z_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/z_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1
for c in cfg2 cfg1 cfg3 cfg4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/z_bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/z_bench_$c.log
done
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu > gpurun_out/z_bench_cfg5.log 2>&1; echo "rc=$?" >> gpurun_out/z_bench_cfg5.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/z_launches_cfg2.csv python tools/prof_one.py 65536,64,1 2 > /dev/null 2>&1
