#!/bin/bash
# round-2 first GPU pass: env, chain microbench, full gpu suite, smoke, pair vs no-pair timing, bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/env.txt
nproc >> gpurun_out/env.txt
timeout 120 ./tools/chain2_bench > gpurun_out/chain2.log 2>&1
for lib in paper_2509_03015_b200/libblocktri_b200.so tools/lib_nopair.so; do
  echo "== $lib" >> gpurun_out/pair_time.log
  BTD_LIB=$lib timeout 300 python tools/quick_time.py 65536,64,1 131072,64,4 20000,48,2 1024,32,1 >> gpurun_out/pair_time.log 2>&1
  BTD_LIB=$lib timeout 300 python tools/level_times.py 65536,64,1 1024,32,1 >> gpurun_out/pair_time.log 2>&1
done
timeout 2400 python -m pytest tests -q -m gpu --durations=15 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.log 2>&1
echo "rc=$?" >> gpurun_out/bench_default.log
