# full validation + bench lines + launch list for profiles/
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_cfg2.log
for c in cfg1 cfg3 cfg4; do timeout -s KILL 900 python bench.py --no-cpu --config $c > gpurun_out/bench_$c.log 2>&1; echo $c=$?; tail -1 gpurun_out/bench_$c.log; done
timeout -s KILL 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?; tail -1 gpurun_out/bench_ref.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python tools/prof_one.py 65536,64,1 > /dev/null 2>&1; echo ncu=$?
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python tools/prof_one.py 1048576,8,1 > /dev/null 2>&1; echo ncu3=$?
