timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 300 python tools/prof_levels.py 1048576,8,1 | tail -1
for v in sm3 sm5; do BTD_LIB=tools/libblocktri_b200_$v.so timeout -s KILL 300 python tools/prof_levels.py 1048576,8,1 | tail -1; done
