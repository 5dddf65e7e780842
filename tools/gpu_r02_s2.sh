python tools/host_micro.py 1024,32,1 > gpurun_out/t2_host_micro.log 2>&1
python bench.py --config cfg1 --steps 50 --warmup 5 > gpurun_out/t2_bench_cfg1.log 2>&1
