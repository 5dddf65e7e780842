#!/bin/bash
# pair-slot level kernel: chain microbenchmark, parity subset, A/B timing vs factor_level_kernel
mkdir -p gpurun_out
./tools/chain2_bench > gpurun_out/chain2.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graphs.py -q -x -k "not baseline_configs" > gpurun_out/pair_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/pair_pytest.log
for lib in paper_2509_03015_b200/libblocktri_b200.so tools/lib_nopair.so tools/lib_r1.so; do
  echo "== $lib" >> gpurun_out/pair_time.log
  BTD_LIB=$lib timeout 600 python tools/quick_time.py 65536,64,1 131072,64,4 20000,48,2 1024,32,1 >> gpurun_out/pair_time.log 2>&1
  BTD_LIB=$lib timeout 600 python tools/level_times.py 65536,64,1 >> gpurun_out/pair_time.log 2>&1
done
