#!/bin/bash
# n = 128 NPD probe (hang hunt), small-block v2 kernels: parity + A/B timing, pair phase profile, Kalman on seam kernels
mkdir -p gpurun_out
for c in one_tile1 one_tile0 two halfB; do
  for g in 1 0; do
    BTD_GRAPHS=$g CUDA_LAUNCH_BLOCKING=1 timeout 60 python tools/npd_probe.py $c >> gpurun_out/c_npd_probe.log 2>&1; echo "$c graphs=$g rc=$?" >> gpurun_out/c_npd_probe.log
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graphs.py -q -x -p no:cacheprovider -k "not bad6 and not bad7" > gpurun_out/c_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c_pytest.log
for lib in paper_2509_03015_b200/libblocktri_b200.so tools/lib_s2_3.so tools/lib_s1.so; do
  echo "== $lib" >> gpurun_out/c_time.log
  BTD_LIB=$lib timeout 300 python tools/quick_time.py 1048576,8,1 200000,5,2 >> gpurun_out/c_time.log 2>&1
  BTD_LIB=$lib timeout 300 python tools/level_times.py 1048576,8,1 >> gpurun_out/c_time.log 2>&1
done
BTD_PROF_LIB=tools/lib_pair_prof.so timeout 300 python tools/phase_prof.py 65536,64,1 > gpurun_out/c_pair_phase.log 2>&1
timeout 600 python -m pytest tests/test_kalman_golden.py tests/test_gpu_seam.py tests/test_gpu_dropin_api.py -q -p no:cacheprovider > gpurun_out/c_kalman.log 2>&1; echo "rc=$?" >> gpurun_out/c_kalman.log
timeout 300 python tools/bench_kalman.py --horizon 100 --state 256 --obs 1024 > gpurun_out/c_kalman_paper.log 2>&1
