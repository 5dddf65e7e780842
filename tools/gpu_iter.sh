timeout -s KILL 600 python -m pytest tests/test_kalman_golden.py -x -q 2>&1 | tail -15
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
