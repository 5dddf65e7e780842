#!/bin/bash
mkdir -p gpurun_out
for c in 512,128,1 256,256,1; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_launches_$c.csv python tools/prof_one.py $c 1 > /dev/null 2>&1
done
timeout 300 python tools/quick_time.py 512,128,1 256,256,1 2048,128,1 > gpurun_out/l_time.log 2>&1
