# iteration loop: parity tests, quick timing, per-level factor times
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
python tools/quick_time.py 65536,64,1 1024,32,1 1048576,8,1 2>&1 | tail -3
python tools/prof_levels.py 65536,64,1 2>&1 | tail -1
