# DRAM traffic per launch of the step's main kernels: ncu --set full with the default
# cache control (L2 flushed before each replay pass), graph replays; CSV export
mkdir -p gpurun_out/ncu_cold
for spec in "k_fchain|chain_kernel<0,.1,.2>|2" "k_bchain|chain_kernel<3,.4,.5>|2" "k_l2|TcRed<.*L2Prob>|8" "k_l3|TcRed<.*L3Prob>|8" "k_l6|TcRed<.*L6Prob>|8" "k_l10|TcRed<.*L10Prob>|8" "k_l7|TcRow<.*L7Prob>|8" "k_msg|TcRow<.*MsgProb>|8" "k_agg|agg4_kernel|8" "k_seg|seg2v_kernel|10" "k_a1|edge_a1_kernel|8" "k_prep|edge_bwd_prep|8" "k_col|colsum2_kernel|10" "k_fdx|TcRow<.*FDxSfProb>|2" "k_fgrad|TcRed<.*FGradProb>|2" "k_force|TcRow<.*ForceProb>|2" "k_af0|edge_af0_kernel|2"; do
  IFS='|' read -r n r k <<< "$spec"
  timeout 600 ncu --set full --clock-control none --kernel-name-base demangled \
    -k "regex:$r" -s "$k" -c 1 -f -o "/tmp/$n" python tools/profile_step.py --steps 3 --graph > "gpurun_out/ncu_cold/$n.log" 2>&1
  echo "$n rc=$?"
  ncu -i "/tmp/$n.ncu-rep" --page raw --csv > "gpurun_out/ncu_cold/$n.raw.csv" 2>/dev/null
  ncu -i "/tmp/$n.ncu-rep" --page details --csv > "gpurun_out/ncu_cold/$n.details.csv" 2>/dev/null
done
