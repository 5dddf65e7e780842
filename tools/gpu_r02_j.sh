#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/quick_time.py 1048576,8,1 200000,5,2 300000,8,4 1024,32,1 > gpurun_out/j_time.log 2>&1
timeout 300 python tools/level_times.py 1048576,8,1 1024,32,1 >> gpurun_out/j_time.log 2>&1
BTD_PROF_LIB=tools/lib_prof.so timeout 300 python tools/phase_prof.py 1024,32,1 20000,32,1 > gpurun_out/j_phase.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -n 1 -p no:cacheprovider > gpurun_out/j_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/j_pytest.log
