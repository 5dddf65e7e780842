#!/bin/bash
mkdir -p gpurun_out
for lib in paper_2509_03015_b200/libblocktri_b200.so tools/lib_skt.so; do
  echo "== $lib" >> gpurun_out/e2_time.log
  BTD_LIB=$lib timeout 300 python tools/quick_time.py 4096,256,64 256,256,1 512,128,4 1024,256,16 >> gpurun_out/e2_time.log 2>&1
done
BTD_LIB=tools/lib_skt.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "sweep or cfg4" > gpurun_out/e2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e2_pytest.log
