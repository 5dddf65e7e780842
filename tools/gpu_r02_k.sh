#!/bin/bash
mkdir -p gpurun_out
timeout 120 ./tools/chain2_bench > gpurun_out/k_chain2.log 2>&1
for lib in paper_2509_03015_b200/libblocktri_b200.so tools/lib_prev.so; do
  echo "== $lib" >> gpurun_out/k_time.log
  BTD_LIB=$lib timeout 300 python tools/quick_time.py 65536,64,1 1024,32,1 20000,48,2 >> gpurun_out/k_time.log 2>&1
  BTD_LIB=$lib timeout 300 python tools/level_times.py 65536,64,1 1024,32,1 >> gpurun_out/k_time.log 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graphs.py -q -x -p no:cacheprovider > gpurun_out/k_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k_pytest.log
