python tools/level_times.py 4096,256,64 512,128,8 > gpurun_out/b3_levels.log 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_graphs.py -m gpu -x -q > gpurun_out/b3_pytest.log 2>&1
python bench.py --config cfg4 --steps 5 --warmup 3 > gpurun_out/b3_bench_cfg4.log 2>&1
