set -x
python -m pytest tests/test_gpu_seam.py tests/test_gpu_dropin_api.py tests/test_kalman_golden.py -m gpu -x -q > gpurun_out/n2_pytest.log 2>&1
python tools/prof_kalman.py > gpurun_out/n2_prof.log 2>&1
python tools/bench_kalman.py --horizon 100 --state 256 --obs 1024 > gpurun_out/n2_kalman_paper.log 2>&1
