#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "sweep or cfg4 or multi or golden or host" > gpurun_out/f2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f2_pytest.log
for lib in paper_2509_03015_b200/libblocktri_b200.so tools/lib_nodm.so; do
  echo "== $lib" >> gpurun_out/f2_time.log
  BTD_LIB=$lib timeout 300 python tools/quick_time.py 4096,256,64 1024,256,16 512,128,8 2048,128,64 >> gpurun_out/f2_time.log 2>&1
done
