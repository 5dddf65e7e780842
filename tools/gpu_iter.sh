timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 300 python tools/quick_time.py 4096,256,64 600,128,3 | tail -2
