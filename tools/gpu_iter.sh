mkdir -p gpurun_out
timeout -s KILL 200 compute-sanitizer --tool memcheck python tools/debug_small.py 2>&1 | grep -E "ERROR SUMMARY|Invalid|^[0-9]+ " | head -20
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -3
timeout -s KILL 200 python tools/quick_time.py 1048576,8,1 1000000,5,2 | tail -2
BTD_SMALL=0 timeout -s KILL 200 python tools/quick_time.py 1048576,8,1 | tail -1
timeout -s KILL 200 python tools/prof_levels.py 1048576,8,1 | tail -1
BTD_LIB=tools/libblocktri_b200_sm4.so timeout -s KILL 200 python tools/quick_time.py 1048576,8,1 | tail -1
