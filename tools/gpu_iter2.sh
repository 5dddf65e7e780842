mkdir -p gpurun_out
timeout -s KILL 120 python tools/phase_prof.py 64,64,1,64 2>&1 | tail -1
