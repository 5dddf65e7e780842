#!/bin/bash
# config 5 on one GPU: unsharded vs sharded (run_sharded_local G=2/4/8), the N=1 bench line, and
# the N=2 bench (two ranks on one GPU over gloo: the multi-rank path end to end)
mkdir -p gpurun_out
timeout 900 python tools/cfg5_check.py > gpurun_out/cfg5_check.log 2>&1; echo "rc=$?" >> gpurun_out/cfg5_check.log
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_cfg5_n1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg5_n1.log
BTD_BENCH_GLOO=1 timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_cfg5_n2_gloo.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg5_n2_gloo.log
