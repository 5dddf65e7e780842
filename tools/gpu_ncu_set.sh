# ncu --set full captures (one launch each) of the dominant kernels of cfg2, cfg3 and cfg4; raw pages
# exported as CSV for tools/ncu_summary.py
mkdir -p gpurun_out
cap() {  # name regex cfg [skip]
  ncu --set full --clock-control none -k regex:$2 -s ${4:-0} -c 1 -o /tmp/ncu_$1 -f python tools/prof_one.py $3 > gpurun_out/ncu_$1.log 2>&1
  ncu -i /tmp/ncu_$1.ncu-rep --page raw --csv > gpurun_out/ncu_$1_raw.csv 2>&1
  echo $1=$?
}
cap cfg2_factor_l0 factor_level_kernel 65536,64,1
cap cfg2_solve_l0 solve_tma_kernel 65536,64,1
cap cfg3_factor_l0 factor_small_kernel 1048576,8,1
cap cfg3_solve_l0 solve_small_kernel 1048576,8,1
cap cfg4_gemm bt_gemm_kernel 4096,256,64 3
cap cfg4_potrf big_potrf_kernel 4096,256,64
