#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/quick_time.py 65536,64,1 1024,64,1 > gpurun_out/o_time.log 2>&1
timeout 300 python tools/level_times.py 65536,64,1 >> gpurun_out/o_time.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graphs.py -q -x -p no:cacheprovider > gpurun_out/o_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/o_pytest.log
BTD_GRAPHS=0 timeout 1500 compute-sanitizer --tool racecheck --print-limit 400 python tools/sanitize_small.py > gpurun_out/o_racecheck.log 2>&1
echo "rc=$?" >> gpurun_out/o_racecheck.log
