#!/bin/bash
mkdir -p gpurun_out
for lib in paper_2509_03015_b200/libblocktri_b200.so tools/lib_prev.so; do
  echo "== $lib" >> gpurun_out/t_time.log
  BTD_LIB=$lib timeout 300 python tools/quick_time.py 65536,64,1 1024,64,1 20000,48,2 >> gpurun_out/t_time.log 2>&1
  BTD_LIB=$lib timeout 300 python tools/level_times.py 65536,64,1 >> gpurun_out/t_time.log 2>&1
done
BTD_PROF_LIB=tools/lib_prof.so timeout 300 python tools/phase_prof.py 65536,64,1 > gpurun_out/t_phase.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graphs.py -q -x -p no:cacheprovider > gpurun_out/t_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t_pytest.log
