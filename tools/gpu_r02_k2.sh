set -x
python tools/prof_kalman.py > gpurun_out/k2_prof.log 2>&1
python tools/bench_kalman.py --horizon 100 --state 256 --obs 1024 > gpurun_out/k2_kalman_paper.log 2>&1
