#!/bin/bash
# cluster-resident serial base for n = 128..256
mkdir -p gpurun_out
timeout 300 python tools/quick_time.py 512,128,1 256,256,1 2048,128,1 4096,256,64 > gpurun_out/p_time.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "sweep or npd or golden or cfg4 or schur" > gpurun_out/p_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p_pytest.log
BTD_GRAPHS=0 timeout 1500 compute-sanitizer --tool racecheck --print-limit 400 python tools/sanitize_small.py > gpurun_out/p_racecheck.log 2>&1
echo "rc=$?" >> gpurun_out/p_racecheck.log
BTD_GRAPHS=0 timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_small.py > gpurun_out/p_memcheck.log 2>&1
echo "rc=$?" >> gpurun_out/p_memcheck.log
