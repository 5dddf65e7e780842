mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -3
timeout -s KILL 200 python tools/quick_time.py 1048576,8,1 1024,32,1 65536,64,1 | tail -3
