#!/bin/bash
mkdir -p gpurun_out
for lib in paper_2509_03015_b200/libblocktri_b200.so tools/lib_s2_3.so; do
  echo "== $lib" >> gpurun_out/i_time.log
  BTD_LIB=$lib timeout 300 python tools/quick_time.py 1048576,8,1 200000,5,2 300000,8,4 >> gpurun_out/i_time.log 2>&1
  BTD_LIB=$lib timeout 300 python tools/level_times.py 1048576,8,1 >> gpurun_out/i_time.log 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graphs.py tests/test_gpu_dropin_api.py tests/test_gpu_seam.py tests/test_kalman_golden.py -q -x -p no:cacheprovider > gpurun_out/i_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/i_pytest.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/i_launches_cfg4.csv python tools/prof_one.py 4096,256,64 1 > /dev/null 2>&1
