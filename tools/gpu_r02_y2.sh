python tools/level_times.py 4096,256,64 65536,64,1 > gpurun_out/y2_levels.log 2>&1
python -m pytest tests/test_gpu_graphs.py tests/test_gpu_dropin_api.py -m gpu -x -q > gpurun_out/y2_pytest.log 2>&1
python bench.py --config cfg4 --steps 5 --warmup 3 > gpurun_out/y2_bench_cfg4.log 2>&1
