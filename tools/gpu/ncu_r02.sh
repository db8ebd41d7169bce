# round-2 evidence: launch list of graph-replayed steps (cold, serialised by ncu) + one
# ncu --set full capture per main kernel family (graph step instance), CSV pages under gpurun_out/ncu
mkdir -p gpurun_out/ncu
python tools/profile_step.py --steps 3 --graph > gpurun_out/ncu/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/ncu/launches.csv python tools/profile_step.py --steps 3 --graph > gpurun_out/ncu/launch.log 2>&1
echo "launch list rc=$?"
SPECS="msg|tc_row_kernel.*MsgProb|4 l7a|tc_row_kernel.*L7AsyncProb|4 chainf|chain_kernel<0, 1, 2|3 chainb|chain_kernel<3, 4, 5|3 l6|tc_red_tma_kernel.*L6Prob|4 fgrad|tc_red_tma_kernel.*FGradProb|1 seg2v|seg2v_kernel|5 agg4|agg4_kernel|4 a1|edge_a1_kernel|4 fdx|tc_row_kernel.*FDxSfProb|1 force|tc_row_kernel.*ForceProb|1 l10|tc_red_kernel.*L10Prob|4"
for spec in $SPECS; do
  IFS='|' read -r n r k <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$r" -s "$k" -c 1 -f -o "gpurun_out/ncu/$n" python tools/profile_step.py --steps 3 --graph > "gpurun_out/ncu/$n.log" 2>&1
  echo "$n rc=$?"
  ncu -i "gpurun_out/ncu/$n.ncu-rep" --page raw --csv > "gpurun_out/ncu/$n.raw.csv" 2>/dev/null
  rm -f "gpurun_out/ncu/$n.ncu-rep"
done
du -sh gpurun_out/ncu
