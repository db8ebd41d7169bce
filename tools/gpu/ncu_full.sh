# ncu --set full captures of the step's main kernel families (one instance each, step 2),
# exported to CSV on the box (the .ncu-rep files are too large to bring back)
mkdir -p gpurun_out/ncu
run() {  # name regex skip
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$2" -s "$3" -c 1 -f -o "/tmp/$1" python tools/profile_step.py --steps 2 > "gpurun_out/ncu/$1.log" 2>&1
  echo "$1 rc=$?"
  ncu -i "/tmp/$1.ncu-rep" --page raw --csv > "gpurun_out/ncu/$1.raw.csv" 2>/dev/null
  ncu -i "/tmp/$1.ncu-rep" --page details --csv > "gpurun_out/ncu/$1.details.csv" 2>/dev/null
  ncu -i "/tmp/$1.ncu-rep" --page source --csv > "gpurun_out/ncu/$1.source.csv" 2>/dev/null
}
for spec in ${NCU_SPECS:-"node_row_P|TcRow<.*PProb>|4" "edge_row_L7|TcRow<.*L7Prob>|4" "edge_row_msg|TcRow<.*MsgProb>|4" "edge_red_L6|TcRed<.*L6Prob>|4" "node_red_L2|TcRed<.*L2Prob>|4" "agg4|agg4_kernel|4" "seg2v|seg2v_kernel|5" "bwd_prep|edge_bwd_prep|4" "split_red|split_reduce_kernel|20"}; do
  IFS='|' read -r n r k <<< "$spec"
  run "$n" "$r" "$k"
done
du -sh gpurun_out/ncu
