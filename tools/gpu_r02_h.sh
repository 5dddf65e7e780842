#!/bin/bash
mkdir -p gpurun_out
for lib in paper_2509_03015_b200/libblocktri_b200.so tools/lib_s2_3.so; do
  echo "== $lib" >> gpurun_out/h_time.log
  BTD_LIB=$lib timeout 300 python tools/quick_time.py 1048576,8,1 200000,5,2 >> gpurun_out/h_time.log 2>&1
  BTD_LIB=$lib timeout 300 python tools/level_times.py 1048576,8,1 >> gpurun_out/h_time.log 2>&1
done
