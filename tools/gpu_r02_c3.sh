python -m pytest tests/test_gpu_seam.py tests/test_kalman_golden.py tests/test_gpu_dropin_api.py -m gpu -x -q > gpurun_out/c3_pytest.log 2>&1
python tools/sanitize_seam.py > gpurun_out/c3_seam_plain.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_seam.py > gpurun_out/c3_seam_racecheck.log 2>&1
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_seam.py > gpurun_out/c3_seam_memcheck.log 2>&1
python tools/prof_kalman.py > gpurun_out/c3_prof.log 2>&1
python tools/bench_kalman.py --horizon 100 --state 256 --obs 1024 > gpurun_out/c3_kalman_paper.log 2>&1
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:seam_ --csv --log-file gpurun_out/c3_seam_launches.csv python tools/prof_kalman.py > /dev/null 2>&1
