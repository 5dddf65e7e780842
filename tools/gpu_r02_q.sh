#!/bin/bash
mkdir -p gpurun_out
BTD_PROF_LIB=tools/lib_prof.so timeout 300 python tools/phase_prof.py 256,256,1 > gpurun_out/q_phase.log 2>&1
BTD_PROF_LIB=tools/lib_prof.so timeout 300 python tools/phase_prof.py 512,128,1 >> gpurun_out/q_phase.log 2>&1
timeout 300 python tools/quick_time.py 512,128,1 256,256,1 > gpurun_out/q_time.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "sweep or npd or golden or cfg4" > gpurun_out/q_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q_pytest.log
