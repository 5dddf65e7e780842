#!/bin/bash
# round-2 GPU check: environment facts, the gpu test suite, smoke
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/env.txt
free -g >> gpurun_out/env.txt; nproc >> gpurun_out/env.txt
timeout 2400 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
