#!/bin/bash
# d = 4 solve on all consumer warps: parity sweep, then timings
mkdir -p gpurun_out
rm -f gpurun_out/w_split.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "sweep or baseline or sharded" > gpurun_out/w_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/w_pytest.log
for c in 65536,64,4 65536,64,8 1048576,64,4; do
  echo "== $c" >> gpurun_out/w_split.log
  timeout 600 python tools/prof_dev.py $c 3 >> gpurun_out/w_split.log 2>&1
done
