mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -4
timeout -s KILL 300 python tools/e2e_probe.py
for s in 2 3; do BTD_LIB=tools/libblocktri_b200_s$s.so timeout -s KILL 200 python tools/quick_time.py 65536,64,1 | tail -1; done
timeout -s KILL 200 python tools/quick_time.py 65536,64,1 | tail -1
