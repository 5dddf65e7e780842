python tools/trace_steps.py 1024,32,1 3 > gpurun_out/r2_trace_cfg1.log 2>&1
python tools/trace_steps.py 65536,64,1 2 > gpurun_out/r2_trace_cfg2.log 2>&1
