#!/bin/bash
# two-CTA solve for d > 1: parity sweep, then timings (cfg2-size d = 1/2/4, cfg5)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "sweep or baseline or sharded" > gpurun_out/w_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/w_pytest.log
for c in 65536,64,1 65536,64,2 65536,64,4 65536,64,8 1048576,64,4; do
  echo "== $c" >> gpurun_out/w_split.log
  timeout 600 python tools/prof_dev.py $c 3 >> gpurun_out/w_split.log 2>&1
done
