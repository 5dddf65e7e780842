#!/bin/bash
# config 5 at N=1: factor/solve split (device-generated instance) and its launch list
mkdir -p gpurun_out
timeout 600 python tools/prof_dev.py 1048576,64,4 4 > gpurun_out/c5_split.log 2>&1; echo "rc=$?" >> gpurun_out/c5_split.log
timeout 600 python tools/prof_dev.py 65536,64,4 4 >> gpurun_out/c5_split.log 2>&1
timeout 600 python tools/prof_dev.py 65536,64,1 4 >> gpurun_out/c5_split.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python tools/prof_dev.py 1048576,64,4 1 > /dev/null 2>&1
