# ncu --set full captures of the step's main kernel families (one instance each, step 2)
mkdir -p gpurun_out/ncu
run() {  # name regex skip
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$2" -s "$3" -c 1 -f -o "gpurun_out/ncu/$1" python tools/profile_step.py --steps 2 > "gpurun_out/ncu/$1.log" 2>&1
  echo "$1 rc=$?"
}
run node_row_P   'TcRow<.*PProb>'      4
run edge_row_L7  'TcRow<.*L7Prob>'     4
run edge_row_msg 'TcRow<.*MsgProb>'    4
run edge_red_L6  'TcRed<.*L6Prob>'     4
run node_red_L2  'TcRed<.*L2Prob>'     4
run agg4         'agg4_kernel'         4
run seg2v        'seg2v_kernel'        5
run bwd_prep     'edge_bwd_prep'       4
run split_red    'split_reduce_kernel' 20
ls -la gpurun_out/ncu
