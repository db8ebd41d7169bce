# tensor-pipe utilisation and DRAM traffic of every tensor-core GEMM launch of a graph step
# (one ncu pass over the tc_row / tc_red / chain kernels; metrics only)
mkdir -p gpurun_out/final
python tools/profile_step.py --steps 3 --graph > gpurun_out/final/plain_ps2.log 2>&1 || { echo "plain failed"; exit 1; }
timeout 1200 ncu --clock-control none --kernel-name-base demangled -k "regex:tc_row_kernel|tc_red|chain_kernel" -c 400 \
  --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size \
  --csv --log-file gpurun_out/final/gemms.csv python tools/profile_step.py --steps 3 --graph > gpurun_out/final/ncu_gemms.log 2>&1
echo "ncu rc=$?"
