python tools/level_times.py 65536,64,1 65536,64,1 1048576,64,4 > gpurun_out/v2_levels.log 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/v2_bench_cfg2.log 2>&1
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "64" > gpurun_out/v2_pytest.log 2>&1
