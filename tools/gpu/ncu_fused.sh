# ncu --set full of chosen step kernels (one instance each) + raw/details/source(SASS and CUDA) pages as CSV.
#   NCU_SPECS="name|demangled-name regex|launches to skip ..." bash tools/gpu/ncu_fused.sh
mkdir -p gpurun_out/ncu
python tools/profile_step.py --steps 2 > gpurun_out/ncu/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
SPECS=${NCU_SPECS:-"msgseg|MsgSegProb|0 l7seg|L7SegProb|0"}
for spec in $SPECS; do
  IFS='|' read -r n r k <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$r" -s "$k" -c 1 -f -o "gpurun_out/ncu/$n" python tools/profile_step.py --steps 2 > "gpurun_out/ncu/$n.log" 2>&1
  echo "$n rc=$?"
  ncu -i "gpurun_out/ncu/$n.ncu-rep" --page raw --csv > "gpurun_out/ncu/$n.raw.csv" 2>/dev/null
  ncu -i "gpurun_out/ncu/$n.ncu-rep" --page details --csv > "gpurun_out/ncu/$n.details.csv" 2>/dev/null
  ncu -i "gpurun_out/ncu/$n.ncu-rep" --page source --csv > "gpurun_out/ncu/$n.source.csv" 2>/dev/null
  ncu -i "gpurun_out/ncu/$n.ncu-rep" --page source --print-source cuda --csv > "gpurun_out/ncu/$n.cuda.csv" 2>/dev/null
done
du -sh gpurun_out/ncu
