#!/bin/bash
# full gpu suite + timings after: small-block v2 only, CTA-uniform entry exits, vectorized Linv/L_sub stores
mkdir -p gpurun_out
timeout 300 python tools/quick_time.py 65536,64,1 1048576,8,1 1024,32,1 > gpurun_out/f_time.log 2>&1
timeout 300 python tools/level_times.py 65536,64,1 1048576,8,1 >> gpurun_out/f_time.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -n 1 -p no:cacheprovider --durations=15 > gpurun_out/f_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 300 python tools/bench_kalman.py --horizon 100 --state 256 --obs 1024 > gpurun_out/f_kalman_paper.log 2>&1
