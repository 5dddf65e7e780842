#!/bin/bash
# d = 1 solve variants: parity sweep, then timings
mkdir -p gpurun_out
rm -f gpurun_out/d1_split.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "sweep or baseline or sharded or golden" > gpurun_out/d1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/d1_pytest.log
for c in 65536,64,1 65536,64,4 1048576,64,4; do
  echo "== $c" >> gpurun_out/d1_split.log
  timeout 600 python tools/prof_dev.py $c 3 >> gpurun_out/d1_split.log 2>&1
done
