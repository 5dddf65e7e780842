# iteration loop: parity tests, quick timing, per-level factor times
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -4
timeout -s KILL 300 python tools/quick_time.py 65536,64,1 1024,32,1 2>&1 | tail -2
timeout -s KILL 300 python tools/prof_levels.py 65536,64,1 2>&1 | tail -1
BTD_STREAM=1 timeout -s KILL 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
