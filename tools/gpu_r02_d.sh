#!/bin/bash
# level2 kernel (TRSM against L, inverse off the critical path) + small v2 + CTA-uniform exits
mkdir -p gpurun_out
for c in one_tile0 two; do
  BTD_GRAPHS=1 timeout 60 python tools/npd_probe.py $c >> gpurun_out/d_npd_probe.log 2>&1; echo "$c rc=$?" >> gpurun_out/d_npd_probe.log
done
for lib in paper_2509_03015_b200/libblocktri_b200.so tools/lib_level1.so tools/lib_s1.so; do
  echo "== $lib" >> gpurun_out/d_time.log
  BTD_LIB=$lib timeout 300 python tools/quick_time.py 65536,64,1 20000,48,2 1048576,8,1 200000,5,2 >> gpurun_out/d_time.log 2>&1
  BTD_LIB=$lib timeout 300 python tools/level_times.py 65536,64,1 1048576,8,1 >> gpurun_out/d_time.log 2>&1
done
timeout 1500 python -m pytest tests -q -x -m gpu -p no:cacheprovider --durations=10 > gpurun_out/d_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/d_pytest.log
