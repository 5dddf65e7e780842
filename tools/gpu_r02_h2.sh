#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin_api.py tests/test_gpu_seam.py -q -x -p no:cacheprovider > gpurun_out/h2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/h2_pytest.log
for lib in paper_2509_03015_b200/libblocktri_b200.so tools/lib_prev.so; do
  echo "== $lib" >> gpurun_out/h2_time.log
  BTD_LIB=$lib timeout 300 python tools/quick_time.py 1048576,8,1 200000,5,2 300000,8,4 >> gpurun_out/h2_time.log 2>&1
  BTD_LIB=$lib timeout 300 python tools/level_times.py 1048576,8,1 >> gpurun_out/h2_time.log 2>&1
done
