#!/bin/bash
# full validation + bench lines of the current build (re-entry session)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f_smoke.log
for c in cfg2 cfg1 cfg3; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/f_bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/f_bench_$c.log
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/f_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/f_bench_ref.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_cfg2.csv python tools/prof_one.py 65536,64,1 2 > /dev/null 2>&1
