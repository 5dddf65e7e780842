mkdir -p gpurun_out
BTD_BENCH_GLOO=1 timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_shard2.log 2>&1; echo shard2=$?; tail -3 gpurun_out/bench_shard2.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_cfg2.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_cfg2.log
