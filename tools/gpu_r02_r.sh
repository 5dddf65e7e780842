#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -n 1 -p no:cacheprovider > gpurun_out/r_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r_pytest.log
BTD_GRAPHS=0 timeout 1500 compute-sanitizer --tool racecheck --print-limit 400 python tools/sanitize_small.py > gpurun_out/r_racecheck.log 2>&1
echo "rc=$?" >> gpurun_out/r_racecheck.log
timeout 300 python tools/quick_time.py 65536,64,1 1048576,8,1 4096,256,64 > gpurun_out/r_time.log 2>&1
