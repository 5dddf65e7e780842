mkdir -p gpurun_out
python tools/phase_prof.py 64,64,1,64 65,64,1,64 82,64,1,64 65536,64,1 > gpurun_out/phase.log 2>&1
cat gpurun_out/phase.log
