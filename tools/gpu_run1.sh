set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo bench=$?
tail -2 gpurun_out/bench_cfg2.log
for c in cfg1 cfg3 cfg4; do timeout 600 python bench.py --no-cpu --config $c > gpurun_out/bench_$c.log 2>&1; echo $c=$?; tail -1 gpurun_out/bench_$c.log; done
