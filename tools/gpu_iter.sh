timeout -s KILL 600 python -m pytest tests/test_kalman_golden.py tests/test_btdfile.py -x -q 2>&1 | tail -3
timeout -s KILL 600 python -m pytest tests -m gpu -q 2>&1 | tail -2
