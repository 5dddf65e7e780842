python tools/level_times.py 65536,64,1 65536,64,1 1024,32,1 > gpurun_out/w2_levels.log 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/w2_bench_cfg2.log 2>&1
python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/w2_pytest.log 2>&1
