#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/h2d_bw.py > gpurun_out/n_h2d.log 2>&1
BTD_GRAPHS=0 timeout 1500 compute-sanitizer --tool racecheck --print-limit 400 python tools/sanitize_small.py > gpurun_out/n_racecheck.log 2>&1
echo "rc=$?" >> gpurun_out/n_racecheck.log
timeout 300 python tools/quick_time.py 65536,64,1 1024,32,1 > gpurun_out/n_time.log 2>&1
