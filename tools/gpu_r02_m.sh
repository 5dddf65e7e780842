#!/bin/bash
# compute-sanitizer over every kernel family after the round-2 kernel changes
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  BTD_GRAPHS=0 timeout 1200 compute-sanitizer --tool $tool --print-limit 200 python tools/sanitize_small.py > gpurun_out/m_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/m_$tool.log
done
