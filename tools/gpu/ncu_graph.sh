# ncu --set full of selected kernels inside graph replays (warm L2, like the timed step); CSV export
mkdir -p gpurun_out/ncu
for spec in ${NCU_SPECS}; do
  IFS='|' read -r n r k <<< "$spec"
  timeout 600 ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base demangled \
    -k "regex:$r" -s "$k" -c 1 -f -o "/tmp/$n" python tools/profile_step.py --steps 3 --graph > "gpurun_out/ncu/$n.log" 2>&1
  echo "$n rc=$?"
  ncu -i "/tmp/$n.ncu-rep" --page raw --csv > "gpurun_out/ncu/$n.raw.csv" 2>/dev/null
  ncu -i "/tmp/$n.ncu-rep" --page details --csv > "gpurun_out/ncu/$n.details.csv" 2>/dev/null
  ncu -i "/tmp/$n.ncu-rep" --page source --csv > "gpurun_out/ncu/$n.source.csv" 2>/dev/null
done
