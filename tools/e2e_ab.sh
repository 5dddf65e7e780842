for g in 1 0 1 0; do BTD_GRAPHS=$g python bench.py --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('graphs=$g', d['ms_per_step'], d['e2e']['ms_per_step'], d['factor_ms'], d['solve_ms'])"; done
BTD_LIB=tools/lib_scalarfrag.so python tools/quick_time.py 65536,64,1; python tools/quick_time.py 65536,64,1; BTD_LIB=tools/lib_scalarfrag.so python tools/quick_time.py 65536,64,1; python tools/quick_time.py 65536,64,1
