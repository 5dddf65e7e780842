ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/a3_launches_cfg4.csv python tools/prof_one.py 4096,256,64 1 > /dev/null 2>&1
python tools/level_times.py 4096,256,64 > gpurun_out/a3_levels.log 2>&1
