set -x
python -m pytest tests/test_gpu_seam.py -m gpu -x -q > gpurun_out/p2_pytest.log 2>&1
python tools/level_times.py 1024,32,1 > gpurun_out/p2_levels.log 2>&1
python tools/torch_prof.py 1024,32,1 factor > gpurun_out/p2_tprof_factor.log 2>&1
python tools/torch_prof.py 1024,32,1 solve > gpurun_out/p2_tprof_solve.log 2>&1
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/p2_launches_cfg1.csv python tools/prof_one.py 1024,32,1 1 > /dev/null 2>&1
