#!/bin/bash
mkdir -p gpurun_out
for lib in tools/lib_l2_prof.so tools/lib_l1_prof.so; do
  echo "== $lib" >> gpurun_out/e_phase.log
  BTD_PROF_LIB=$lib timeout 300 python tools/phase_prof.py 65536,64,1 >> gpurun_out/e_phase.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "host_input" > gpurun_out/e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e_pytest.log
