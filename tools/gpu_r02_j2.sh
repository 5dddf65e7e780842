#!/bin/bash
mkdir -p gpurun_out
for lib in paper_2509_03015_b200/libblocktri_b200.so tools/lib_areg.so; do
  echo "== $lib" >> gpurun_out/j2_time.log
  BTD_LIB=$lib timeout 300 python tools/quick_time.py 65536,64,1 20000,48,2 >> gpurun_out/j2_time.log 2>&1
  BTD_LIB=$lib timeout 300 python tools/level_times.py 65536,64,1 >> gpurun_out/j2_time.log 2>&1
done
BTD_LIB=tools/lib_areg.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "golden or sweep or schur or npd or host or device or multi" > gpurun_out/j2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/j2_pytest.log
