timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout -s KILL 200 python tools/quick_time.py 65536,64,1 | tail -1
timeout -s KILL 200 python tools/prof_levels.py 65536,64,1 | tail -1
