#!/bin/bash
# compute-sanitizer on the d > 1 solve paths, plus a verbose GPU-suite run
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  BTD_GRAPHS=0 timeout 1200 compute-sanitizer --tool $tool --kernel-name regex:solve_tma python tools/sanitize_solve4.py > gpurun_out/san4_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/san4_$tool.log
done
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -rA --durations=10 > gpurun_out/i_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/i_pytest.log
