#!/bin/bash
# round 2: chain microbenchmark, n=128 NPD probe, pair-kernel parity subset, A/B timing
mkdir -p gpurun_out
./tools/chain2_bench > gpurun_out/chain2.log 2>&1
for c in one_tile1 one_tile0 two halfB; do
  for g in 1 0; do
    BTD_GRAPHS=$g timeout 60 python tools/npd_probe.py $c >> gpurun_out/npd_probe.log 2>&1; echo "$c graphs=$g rc=$?" >> gpurun_out/npd_probe.log
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graphs.py -v -x -k "not baseline_configs and not 128-8-64" --durations=10 > gpurun_out/pair_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/pair_pytest.log
for lib in paper_2509_03015_b200/libblocktri_b200.so tools/lib_nopair.so tools/lib_r1.so; do
  echo "== $lib" >> gpurun_out/pair_time.log
  BTD_LIB=$lib timeout 300 python tools/quick_time.py 65536,64,1 131072,64,4 20000,48,2 1024,32,1 >> gpurun_out/pair_time.log 2>&1
  BTD_LIB=$lib timeout 300 python tools/level_times.py 65536,64,1 1024,32,1 >> gpurun_out/pair_time.log 2>&1
done
