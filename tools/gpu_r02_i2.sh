#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_sweep.sh > /dev/null 2>&1
cp gpurun_out/sweep.md gpurun_out/i2_sweep.md
