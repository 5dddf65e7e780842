#!/bin/bash
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b2_launches_cfg2.csv python tools/prof_one.py 65536,64,1 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b2_launches_cfg3.csv python tools/prof_one.py 1048576,8,1 1 > /dev/null 2>&1
timeout 300 python tools/quick_time.py 65536,64,1 1048576,8,1 > gpurun_out/b2_time.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -n 1 -p no:cacheprovider > gpurun_out/b2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/b2_pytest.log
