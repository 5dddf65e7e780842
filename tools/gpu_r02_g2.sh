#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "sweep or cfg4 or multi" > gpurun_out/g2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g2_pytest.log
timeout 300 python tools/quick_time.py 4096,256,64 512,128,8 700,128,6 > gpurun_out/g2_time.log 2>&1
