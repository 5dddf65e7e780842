./tools/potrf_bench | tail -2
./tools/panel_bench2
bash tools/gpu_ncu_solve.sh
