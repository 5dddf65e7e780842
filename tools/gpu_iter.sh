timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 300 python tools/quick_time.py 65536,64,1 1024,32,1 20000,64,4 4096,256,64 | tail -4
