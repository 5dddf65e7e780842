set -x
python -m pytest tests -m gpu -x -q > gpurun_out/l2_pytest.log 2>&1
python tools/prof_kalman.py > gpurun_out/l2_prof.log 2>&1
python tools/bench_kalman.py --horizon 100 --state 256 --obs 1024 > gpurun_out/l2_kalman_paper.log 2>&1
python tools/bench_kalman.py > gpurun_out/l2_kalman.log 2>&1
