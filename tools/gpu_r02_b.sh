#!/bin/bash
# round-2: full gpu suite (verbose, crash-tolerant via one xdist worker), the host-input test on the
# pair build, then config 5
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -v -m gpu -n 1 --durations=20 -p no:cacheprovider > gpurun_out/pytest_gpu_v.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_v.log
BTD_LIB=tools/lib_pair.so CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest tests/test_gpu_parity.py -v -x -k "host_input_overlapped" -p no:cacheprovider > gpurun_out/pair_hostinput.log 2>&1
echo "rc=$?" >> gpurun_out/pair_hostinput.log
bash tools/gpu_r02_cfg5.sh
